"""GPU parity for the sharded engine queues with global admission (SURVEY §8f
row 1): the golden EngineSim scripts (enqueue / scheduling_iteration /
completions, written by the unmodified reference) replayed with every
enqueue batch split over G shard schedulers on one device. The Mode B relay
of the engine counters is done by copying them shard to shard; each
scheduling iteration is chm_queue_candidates on every shard, the candidates
stacked (what dist.sharded_iteration all-gathers), then
chm_queue_admit_merged on every shard. Admission order, the union queue's
STJF order, starvation levels / counts, running and iteration counters must
equal the single reference queue."""

import math

import numpy as np
import pytest
import torch

from paper_2603_22206_b200.config import AgingConfig, BalancerConfig, ModelProfile, Pool
from paper_2603_22206_b200.dist import _RELAYED
from paper_2603_22206_b200.predictor import PrecomputedPredictor
from paper_2603_22206_b200.router import ScoreTableRouter
from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch
from tests import harness as H

pytestmark = pytest.mark.gpu


def _key_tuple(k):
    """chm_queue_key int64 words -> the reference sort key (level, priority,
    arrival, seq) and the handle."""
    lv, pb, ab, sq, hd = (int(x) for x in k)
    pr = np.array([pb], dtype=np.int64).view(np.float64)[0]
    ar = np.array([ab], dtype=np.int64).view(np.float64)[0]
    return (lv, float(pr), float(ar), sq), hd


def replay_sharded(qd, G, capacity=10240):
    S = qd["S"] if qd["S"] else math.inf
    pool = Pool((ModelProfile("m0", 1.0, qd["b"]),))
    enq = qd["enq"]
    shards = []
    for _ in range(G):
        rt, pr = ScoreTableRouter(), PrecomputedPredictor()
        aging = AgingConfig(starvation_threshold=S, running_quantum=qd["Q"],
                            demote_while_queued=qd["demote"])
        gs = GpuScheduler(pool, BalancerConfig(), aging, router=rt,
                          predictor=pr, n_programs=len(enq) + 1, max_rows=max(len(enq), 1),
                          queue_capacity=capacity)
        shards.append((gs, rt, pr))
    dev = shards[0][0].device
    admitted = []
    pos = 0

    def relay(src, dst):
        for name in _RELAYED + ("inflight_sum", "inflight_comp"):
            getattr(dst.state, name).copy_(getattr(src.state, name))

    def enqueue(n_rows):
        nonlocal pos
        o = enq[pos:pos + n_rows]
        pos += n_rows
        bounds = np.linspace(0, n_rows, G + 1).astype(int)
        for g, (gs, rt, pr) in enumerate(shards):
            if g > 0:
                relay(shards[g - 1][0], gs)
            part = o[bounds[g]:bounds[g + 1]]
            n = len(part)
            rt.set(torch.full((n, 1), 0.5, dtype=torch.float32, device=dev))
            pr.set(torch.as_tensor(part[:, 1] if n else np.zeros(0), device=dev).reshape(-1, 1))
            b = RowBatch.from_numpy(dev, program=part[:, 0].astype(np.int32), stage=np.ones(n),
                                    arrival=part[:, 2], out_tokens=np.full((n, 1), 10 ** 9),
                                    handle=part[:, 0].astype(np.int64))
            gs.run_rows(b, n_iterations=0)
            gs.check_errors()
            fl = gs.buf.dflags[:n].cpu().numpy()
            admitted.extend(int(x) for x in part[(fl & 2) != 0, 0])
        for gs, _, _ in shards[:-1]:  # the last rank broadcasts the tick-end counters
            relay(shards[-1][0], gs)

    def iteration(release=None):
        for gs, _, _ in shards:
            gs.state.q_n_admitted.zero_()
        gathered = torch.stack([gs.queue_candidates() for gs, _, _ in shards])
        rel = None if release is None else torch.tensor([release], dtype=torch.int32, device=dev)
        for g, (gs, _, _) in enumerate(shards):
            gs.queue_admit_merged(gathered, g, rel)
            gs.check_errors()
        keys = dict(_key_tuple(k)[::-1] for k in gathered.reshape(-1, 5).cpu().numpy())
        new = [int(h) for gs, _, _ in shards for h in gs.state.admitted(0)]
        admitted.extend(sorted(new, key=lambda h: keys[h]))

    enqueue(qd["n_pre"])
    for op, n in qd["script"]:
        if op == "enq":
            enqueue(n)
        elif op == "iter":
            for _ in range(n):
                iteration()
        else:
            for _ in range(n):
                iteration(release=1)
    # union of the sub-queues in the global STJF order
    rows = []
    for gs, _, _ in shards:
        st = gs.state
        nq = int(st.engine_queued[0])
        for i in range(nq):
            key = (int(st.q_level[i]), float(st.q_priority[i]), float(st.q_arrival[i]),
                   int(st.q_seq[i]))
            rows.append((key, int(st.q_handle[i]), int(st.q_count[i])))
    rows.sort()
    runs = {int(gs.state.engine_running[0]) for gs, _, _ in shards}
    iters = {int(gs.state.engine_iterations[0]) for gs, _, _ in shards}
    assert len(runs) == 1 and len(iters) == 1, (runs, iters)
    return dict(
        admitted=np.array(admitted),
        order=np.array([r[1] for r in rows]),
        level=np.array([r[0][0] for r in rows]),
        count=np.array([r[2] for r in rows]),
        running=runs.pop(),
        iterations=iters.pop(),
    )


@pytest.mark.parametrize("capacity", [10240, 20480])  # smem / global-memory keys
@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name", H.queue_names())
def test_sharded_queue_matches_reference(name, G, capacity):
    qd = H.load_queue(name)
    res = replay_sharded(qd, G, capacity)
    np.testing.assert_array_equal(res["admitted"], qd["admitted"])
    np.testing.assert_array_equal(res["order"], qd["order"])
    np.testing.assert_array_equal(res["level"], qd["level"])
    np.testing.assert_array_equal(res["count"], qd["count"])
    assert res["running"] == qd["running"]
    assert res["iterations"] == qd["iterations"]


def test_candidates_report_the_stjf_head():
    """chm_queue_candidates: the first max_batch_size entries in STJF order,
    padded with level = INT64_MAX."""
    qd = H.load_queue("q_basic")
    pool = Pool((ModelProfile("m0", 1.0, 4),))
    rt, pr = ScoreTableRouter(), PrecomputedPredictor()
    gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=8), router=rt,
                      predictor=pr, n_programs=64, max_rows=32)
    dev = gs.device
    o = qd["enq"][:10]
    rt.set(torch.full((10, 1), 0.5, dtype=torch.float32, device=dev))
    pr.set(torch.as_tensor(o[:, 1], device=dev).reshape(-1, 1))
    gs.run_rows(RowBatch.from_numpy(dev, program=o[:, 0].astype(np.int32), stage=np.ones(10),
                                    arrival=o[:, 2], out_tokens=np.full((10, 1), 10 ** 9),
                                    handle=o[:, 0].astype(np.int64)), n_iterations=0)
    gs.check_errors()
    cand = gs.queue_candidates().cpu().numpy()[0]
    head = gs.state.queue_order(0)[:4]
    assert [int(c[4]) for c in cand] == [int(h) for h in head]
    empty = gs.queue_candidates()
    assert empty.shape == (1, 4, 5)
