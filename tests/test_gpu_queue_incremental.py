"""K7 grid-wide queue path over several ticks: the incremental fast path
(stjf_huge.cu: kept STJF order + insertion, in-place compaction, class merge)
against the single-CTA global-key path (pinned to the reference goldens in
test_gpu_queue.py) and against the grid-wide radix path (CHM_QUEUE_FAST=0).

Every tick appends routed rows, completes some running requests and runs
scheduling iterations with S = 3, so calls admit, age and promote (one, two
and more level classes among the survivors)."""

import os

import numpy as np
import pytest
import torch

from paper_2603_22206_b200 import _lib
from paper_2603_22206_b200.config import AgingConfig, BalancerConfig, ModelProfile, Pool
from paper_2603_22206_b200.predictor import PrecomputedPredictor
from paper_2603_22206_b200.router import ScoreTableRouter
from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch

pytestmark = pytest.mark.gpu

B = (64, 16)


def _run(capacity, n, ticks, seed, rows_per_tick=3000, fast=True):
    os.environ["CHM_QUEUE_FAST"] = "1" if fast else "0"
    try:
        rng = np.random.default_rng(seed)
        pool = Pool((ModelProfile("m0", 1.0, B[0]), ModelProfile("m1", 2.0, B[1])))
        n_prog = ticks * rows_per_tick + 16
        gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=3),
                          router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                          n_programs=n_prog, max_rows=rows_per_tick,
                          queue_capacity=capacity)
        st = gs.state
        for m in range(2):
            prio = np.round(rng.lognormal(5, 2, n))
            prio[rng.random(n) < 0.2] = 37.0  # ties
            arr = np.sort(rng.random(n) * 100)
            st.load_queue(m, prio, arr, np.arange(n), np.arange(n) + (m << 40),
                          level=-rng.integers(0, 3, n), count=rng.integers(0, 3, n))
        st.set_engine_counters(running=list(B), seq=[n, n])
        snaps = []
        dev = gs.device
        for t in range(ticks):
            nr = rows_per_tick if t % 3 != 2 else 0  # every third tick: no arrivals
            q = rng.random((nr, 2)).astype(np.float32)
            yhat = np.round(rng.lognormal(5, 2, (nr, 2)))
            yhat[rng.random((nr, 2)) < 0.2] = 37.0
            gs.router.set(torch.as_tensor(q, device=dev))
            gs.predictor.set(torch.as_tensor(yhat, dtype=torch.float64, device=dev))
            prog = np.arange(nr) + t * rows_per_tick
            batch = RowBatch.from_numpy(dev, program=prog.astype(np.int32), stage=np.ones(nr),
                                        arrival=np.full(nr, 100.0 + t),
                                        out_tokens=np.full((nr, 2), 10 ** 6),
                                        handle=(prog + (1 << 50)).astype(np.int64))
            nc = torch.tensor(rng.integers(0, 6, 2), dtype=torch.int32, device=dev)
            gs.run_rows(batch, n_iterations=int(rng.integers(0, 4)), n_complete=nc)
            gs.check_errors(f"tick {t}")
            snaps.append(_snapshot(gs))
        return snaps
    finally:
        os.environ.pop("CHM_QUEUE_FAST", None)


def _snapshot(gs):
    st = gs.state
    out = {"running": st.engine_running.cpu().numpy().copy(),
           "queued": st.engine_queued.cpu().numpy().copy(),
           "iterations": st.engine_iterations.cpu().numpy().copy(),
           "promoted": st.q_n_promoted.cpu().numpy().copy(),
           "unsorted": st.q_arrival_unsorted.cpu().numpy().copy()}
    for m in range(2):
        nq = int(st.engine_queued[m])
        b = m * st.capacity
        out[f"admitted{m}"] = st.admitted(m)
        out[f"order{m}"] = st.q_order[b:b + nq].cpu().numpy()
        for f in ("level", "count", "quantum", "priority", "arrival", "seq", "handle",
                  "out_tokens"):
            out[f"{f}{m}"] = getattr(st, f"q_{f}")[b:b + nq].cpu().numpy()
    return out


def _same(a, b, what):
    assert len(a) == len(b)
    for t, (x, y) in enumerate(zip(a, b)):
        assert x.keys() == y.keys()
        for k in x:
            np.testing.assert_array_equal(x[k], y[k], err_msg=f"{what}: tick {t}, {k}")


def _fast_calls():
    return int(_lib.load().chm_queue_fast_calls())


def test_incremental_matches_single_cta_over_ticks():
    n, ticks = 180000, 8
    small = _run(262144, n, ticks, seed=11)    # single-CTA global-key path
    f0 = _fast_calls()
    huge = _run(300000, n, ticks, seed=11)     # grid-wide, incremental after tick 0
    # two queue calls per tick (completions, tick), counted per engine; only
    # the first call can't run incrementally
    assert _fast_calls() - f0 == 2 * (2 * ticks - 1)
    _same(small, huge, "single-CTA vs incremental")
    assert sum(int(s["promoted"].sum()) for s in huge) > 0
    assert sum(len(s["admitted0"]) + len(s["admitted1"]) for s in huge) > 0


def test_incremental_matches_radix_at_2m():
    n, ticks = 2_000_000, 4
    f0 = _fast_calls()
    fast = _run(2_097_152, n, ticks, seed=3, fast=True)
    assert _fast_calls() - f0 == 2 * (2 * ticks - 1)
    radix = _run(2_097_152, n, ticks, seed=3, fast=False)
    assert _fast_calls() - f0 == 2 * (2 * ticks - 1)
    _same(radix, fast, "radix vs incremental")


def test_incremental_survives_external_queue_edit():
    """A queue rewritten between calls (load_queue) is detected by the state
    hash: the call falls back to the radix path and still matches."""
    pool = Pool((ModelProfile("m0", 1.0, 4),))
    res = []
    f0 = _fast_calls()
    for capacity in (262144, 300000):
        gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=3),
                          router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                          n_programs=16, max_rows=16, queue_capacity=capacity)
        st = gs.state
        rng = np.random.default_rng(7)
        gs.router.set(torch.zeros((0, 1), device=gs.device))
        gs.predictor.set(torch.zeros((0, 1), dtype=torch.float64, device=gs.device))
        empty = RowBatch.from_numpy(gs.device, program=np.zeros(0), stage=np.zeros(0),
                                    arrival=np.zeros(0), out_tokens=np.zeros((0, 1)),
                                    handle=np.zeros(0))
        snaps = []
        for k in range(3):
            n = 50000 + 1000 * k
            st.load_queue(0, np.round(rng.lognormal(5, 2, n)), np.sort(rng.random(n)),
                          np.arange(n), np.arange(n), level=-rng.integers(0, 2, n),
                          count=rng.integers(0, 3, n))
            st.set_engine_counters(running=[2], seq=[n])
            gs.run_rows(empty, n_iterations=2, n_complete=torch.tensor([1], dtype=torch.int32,
                                                                       device=gs.device))
            gs.check_errors()
            s = {"admitted": st.admitted(0), "queued": int(st.engine_queued[0])}
            s["order"] = st.q_order[:s["queued"]].cpu().numpy()
            s["level"] = st.q_level[:s["queued"]].cpu().numpy()
            snaps.append(s)
        res.append(snaps)
    # per load: the completions call re-sorts (edited queue), the tick continues
    assert _fast_calls() - f0 == 3
    for a, b in zip(*res):
        assert a["queued"] == b["queued"]
        for k in ("admitted", "order", "level"):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.parametrize("fast", [True, False])
def test_graph_replay_matches_eager(fast):
    """The grid-wide path captured in a CUDA graph (its two radix sections as
    IF nodes whose conditions the device sets) replays the eager ticks."""
    from paper_2603_22206_b200.tick import TickGraph

    os.environ["CHM_QUEUE_FAST"] = "1" if fast else "0"
    try:
        rng = np.random.default_rng(5)
        pool = Pool((ModelProfile("m0", 1.0, B[0]), ModelProfile("m1", 2.0, B[1])))
        gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=3),
                          router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                          n_programs=16, max_rows=16, queue_capacity=300000)
        st = gs.state
        n = 180000
        for m in range(2):
            prio = np.round(rng.lognormal(5, 2, n))
            prio[rng.random(n) < 0.2] = 37.0
            st.load_queue(m, prio, np.sort(rng.random(n) * 100), np.arange(n),
                          np.arange(n) + (m << 40), level=-rng.integers(0, 3, n),
                          count=rng.integers(0, 3, n))
        st.set_engine_counters(running=list(B), seq=[n, n])
        dev = gs.device
        gs.router.set(torch.zeros((0, 2), device=dev))
        gs.predictor.set(torch.zeros((0, 2), dtype=torch.float64, device=dev))
        empty = RowBatch.from_numpy(dev, program=np.zeros(0), stage=np.zeros(0),
                                    arrival=np.zeros(0), out_tokens=np.zeros((0, 2)),
                                    handle=np.zeros(0))
        nc = torch.tensor([5, 3], dtype=torch.int32, device=dev)
        snap = st.snapshot()
        eager = []
        for _ in range(5):
            gs.run_rows(empty, n_iterations=2, n_complete=nc)
            gs.check_errors()
            eager.append(_snapshot(gs))
        st.restore(snap)
        tg = TickGraph(gs, empty, n_iterations=2, n_complete=nc)  # warm-up = tick 0, eager
        torch.cuda.synchronize()
        replay = [_snapshot(gs)]
        for _ in range(4):
            tg.replay()
            torch.cuda.synchronize()
            gs.check_errors()
            replay.append(_snapshot(gs))
        _same(eager, replay, "eager vs graph replay")
        assert sum(int(s["promoted"].sum()) for s in eager) > 0
    finally:
        os.environ.pop("CHM_QUEUE_FAST", None)
