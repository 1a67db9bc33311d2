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
    aging = AgingConfig(starvation_threshold=S, running_quantum=qd["Q"],
                        demote_while_queued=qd["demote"])
    gs = GpuScheduler(pool, BalancerConfig(), aging, router=rt,
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


@pytest.mark.parametrize("capacity", [10240, 20480, 300000])  # smem / global keys / grid-wide
@pytest.mark.parametrize("name", H.queue_names())
def test_queue_matches_reference(name, capacity):
    qd = H.load_queue(name)
    if qd["demote"] and capacity > (1 << 18):
        pytest.skip("demote_while_queued runs on the per-engine paths only")
    res = replay_on_gpu(qd, capacity)
    np.testing.assert_array_equal(res["admitted"], qd["admitted"])
    np.testing.assert_array_equal(res["order"], qd["order"])
    np.testing.assert_array_equal(res["level"], qd["level"])
    np.testing.assert_array_equal(res["count"], qd["count"])
    assert res["running"] == qd["running"]
    assert res["iterations"] == qd["iterations"]


def _stress_state(capacity, n, seed, b=(64, 16), S=3):
    """Two engines with n queued entries each: ties, mixed levels/counts, and
    engines with free slots so iterations admit and age at scale."""
    rng = np.random.default_rng(seed)
    pool = Pool((ModelProfile("m0", 1.0, b[0]), ModelProfile("m1", 2.0, b[1])))
    gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=S),
                      router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                      n_programs=16, max_rows=16, queue_capacity=capacity)
    st = gs.state
    for m in range(2):
        prio = np.round(rng.lognormal(5, 2, n))
        prio[rng.random(n) < 0.2] = 37.0  # ties
        arr = np.sort(rng.random(n) * 100)
        st.load_queue(m, prio, arr, np.arange(n), np.arange(n) + (m << 40),
                      level=-rng.integers(0, 3, n), count=rng.integers(0, S, n))
    st.set_engine_counters(running=[b[0] // 2, b[1]])
    gs.router.set(torch.zeros((0, 2), device=gs.device))
    gs.predictor.set(torch.zeros((0, 2), dtype=torch.float64, device=gs.device))
    return gs


def _snapshot_queue(gs):
    st = gs.state
    out = {"running": st.engine_running.cpu().numpy().copy(),
           "queued": st.engine_queued.cpu().numpy().copy(),
           "iterations": st.engine_iterations.cpu().numpy().copy(),
           "promoted": st.q_n_promoted.cpu().numpy().copy()}
    for m in range(2):
        nq = int(st.engine_queued[m])
        b = m * st.capacity
        order = st.q_order[b:b + nq].long()
        out[f"admitted{m}"] = st.admitted(m)
        out[f"order{m}"] = st.q_handle[b:b + nq][order].cpu().numpy()
        for f in ("level", "count", "quantum", "priority", "handle"):
            out[f"{f}{m}"] = getattr(st, f"q_{f}")[b:b + nq].cpu().numpy()
    return out


@pytest.mark.parametrize("n", [150000, 250000])
def test_queue_grid_wide_matches_single_cta(n):
    """The grid-wide path (capacity > 2^18) against the single-CTA global-key
    path (itself pinned to the reference goldens above) on the same state:
    completions, then a tick with 3 iterations (admission + aging + promotion)."""
    res = []
    for capacity in (262144, 300000):
        gs = _stress_state(capacity, n, seed=n)
        e = RowBatch.from_numpy(gs.device, program=np.zeros(0), stage=np.zeros(0),
                                arrival=np.zeros(0), out_tokens=np.zeros((0, 2)),
                                handle=np.zeros(0))
        nc = torch.tensor([5, 3], dtype=torch.int32, device=gs.device)
        gs.run_rows(e, n_iterations=3, n_complete=nc)
        gs.check_errors()
        res.append(_snapshot_queue(gs))
    small, huge = res
    assert small.keys() == huge.keys()
    for k in small:
        np.testing.assert_array_equal(small[k], huge[k], err_msg=k)
    assert small["promoted"].sum() > 0 and len(small["admitted0"]) > 0


@pytest.mark.parametrize("n,capacity", [(9000, 10240), ((9000, 15000), 20480), (70000, 72000),
                                        (2000000, 2097152)])
def test_queue_order_random_large(n, capacity):
    """Full-size STJF order vs a numpy lexsort of (level, priority, arrival, seq);
    70k entries per engine exercises the global-scratch path (cfg4 stress);
    (9000, 15000) at capacity 20480: one CTA keeps its keys in shared memory,
    the other in global scratch (queue_kernel_dual)."""
    ns = n if isinstance(n, tuple) else (n, n)
    rng = np.random.default_rng(5)
    pool = Pool((ModelProfile("m0", 1.0, 4), ModelProfile("m1", 2.0, 4)))
    gs = GpuScheduler(pool, router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                      n_programs=16, max_rows=16, queue_capacity=capacity)
    st = gs.state
    for m in range(2):
        n = ns[m]
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
        n = ns[m]
        b = m * st.capacity
        pr = st.q_priority[b:b + n].cpu().numpy()
        ar = st.q_arrival[b:b + n].cpu().numpy()
        lv = st.q_level[b:b + n].cpu().numpy()
        want = np.lexsort((np.arange(n), ar, pr, lv))
        got = st.q_order[b:b + n].cpu().numpy()
        np.testing.assert_array_equal(got, want)
