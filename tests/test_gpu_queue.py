"""GPU parity for K7 (STJF + aging): replay the golden EngineSim scripts
(enqueue / scheduling_iteration / completions) through the C-ABI and compare
admission order, final queue order, starvation levels and counts."""

import math

import numpy as np
import pytest
import torch

from paper_2603_22206_b200.config import AgingConfig, BalancerConfig, ModelProfile, Pool
from paper_2603_22206_b200.predictor import PrecomputedPredictor
from paper_2603_22206_b200.router import ScoreTableRouter
from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch
from tests import harness as H

pytestmark = pytest.mark.gpu


def replay_on_gpu(qd, capacity=10240):
    S = qd["S"] if qd["S"] else math.inf
    pool = Pool((ModelProfile("m0", 1.0, qd["b"]),))
    rt, pr = ScoreTableRouter(), PrecomputedPredictor()
    enq = qd["enq"]
    gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=S), router=rt,
                      predictor=pr, n_programs=len(enq) + 1, max_rows=max(len(enq), 1),
                      queue_capacity=capacity)
    dev = gs.device
    admitted = []
    pos = 0

    def call(n_rows=0, n_iter=0, n_complete=None):
        nonlocal pos
        o = enq[pos:pos + n_rows]
        pos += n_rows
        rt.set(torch.full((n_rows, 1), 0.5, dtype=torch.float32, device=dev))
        pr.set(torch.as_tensor(o[:, 1] if n_rows else np.zeros(0), device=dev).reshape(-1, 1))
        b = RowBatch.from_numpy(dev, program=o[:, 0].astype(np.int32), stage=np.ones(n_rows),
                                arrival=o[:, 2], out_tokens=np.full((n_rows, 1), 10 ** 9),
                                handle=o[:, 0].astype(np.int64))
        nc = None if n_complete is None else torch.tensor([n_complete], dtype=torch.int32,
                                                          device=dev)
        gs.run_rows(b, n_iterations=n_iter, n_complete=nc)
        gs.check_errors()
        fl = gs.buf.dflags[:n_rows].cpu().numpy()
        admitted.extend(int(x) for x in o[(fl & 2) != 0, 0])
        admitted.extend(int(x) for x in gs.state.admitted(0))

    call(n_rows=qd["n_pre"])
    for op, n in qd["script"]:
        if op == "enq":
            call(n_rows=n)
        elif op == "iter":
            call(n_iter=n)
        else:
            call(n_complete=n)
    st = gs.state
    nq = int(st.engine_queued[0])
    order_idx = st.q_order[:nq].long()
    return dict(
        admitted=np.array(admitted),
        order=st.q_handle[:nq][order_idx].cpu().numpy(),
        level=st.q_level[:nq][order_idx].cpu().numpy(),
        count=st.q_count[:nq][order_idx].cpu().numpy(),
        running=int(st.engine_running[0]),
        iterations=int(st.engine_iterations[0]),
    )


@pytest.mark.parametrize("capacity", [10240, 20480])  # smem keys / global-scratch keys
@pytest.mark.parametrize("name", H.queue_names())
def test_queue_matches_reference(name, capacity):
    qd = H.load_queue(name)
    res = replay_on_gpu(qd, capacity)
    np.testing.assert_array_equal(res["admitted"], qd["admitted"])
    np.testing.assert_array_equal(res["order"], qd["order"])
    np.testing.assert_array_equal(res["level"], qd["level"])
    np.testing.assert_array_equal(res["count"], qd["count"])
    assert res["running"] == qd["running"]
    assert res["iterations"] == qd["iterations"]


@pytest.mark.parametrize("n,capacity", [(9000, 10240), (70000, 72000)])
def test_queue_order_random_large(n, capacity):
    """Full-size STJF order vs a numpy lexsort of (level, priority, arrival, seq);
    70k entries per engine exercises the global-scratch path (cfg4 stress)."""
    rng = np.random.default_rng(5)
    pool = Pool((ModelProfile("m0", 1.0, 4), ModelProfile("m1", 2.0, 4)))
    gs = GpuScheduler(pool, router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                      n_programs=16, max_rows=16, queue_capacity=capacity)
    st = gs.state
    for m in range(2):
        prio = rng.lognormal(5, 2, n)
        prio[rng.random(n) < 0.2] = 37.0  # ties
        arr = np.sort(rng.random(n) * 100)
        lvl = -rng.integers(0, 3, n)
        st.load_queue(m, prio, arr, np.arange(n), np.arange(n) + 1000 * m, level=lvl,
                      count=rng.integers(0, 8, n))
    st.set_engine_counters(running=[4, 4])
    gs.router.set(torch.zeros((0, 2), device=gs.device))
    gs.predictor.set(torch.zeros((0, 2), dtype=torch.float64, device=gs.device))
    e = RowBatch.from_numpy(gs.device, program=np.zeros(0), stage=np.zeros(0),
                            arrival=np.zeros(0), out_tokens=np.zeros((0, 2)), handle=np.zeros(0))
    gs.run_rows(e, n_iterations=0)
    gs.check_errors()
    for m in range(2):
        b = m * st.capacity
        pr = st.q_priority[b:b + n].cpu().numpy()
        ar = st.q_arrival[b:b + n].cpu().numpy()
        lv = st.q_level[b:b + n].cpu().numpy()
        want = np.lexsort((np.arange(n), ar, pr, lv))
        got = st.q_order[b:b + n].cpu().numpy()
        np.testing.assert_array_equal(got, want)
