"""STJF+aging queue stress (N_q up to 16M entries): one engine
with N queued entries (lognormal priorities with ties, mixed starvation
levels / counts), one scheduling tick (admit into free slots + age the rest +
final STJF order) per step, timed with CUDA events around the queue kernels
only (the state is restored between steps, untimed).

  python tools/queue_stress.py [--n 16777216] [--steps 5] [--engines 1] [--chain]

--chain: consecutive ticks on the evolving queue (no restore between steps),
the steady state in which the grid-wide path runs incrementally (a restored
queue no longer matches the state hash the previous call kept, so the default
mode measures the full radix path).

Prints one JSON line per size: ms per tick and achieved GB/s on the
algorithmic bytes (40 B read + 40 B written per entry + 4 B of order) against
MEASURED_PEAKS.json hbm_gbs.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_22206_b200 import _lib  # noqa: E402
from paper_2603_22206_b200.config import AgingConfig, BalancerConfig, ModelProfile, Pool  # noqa: E402
from paper_2603_22206_b200.predictor import PrecomputedPredictor  # noqa: E402
from paper_2603_22206_b200.router import ScoreTableRouter  # noqa: E402
from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch  # noqa: E402

BYTES_PER_ENTRY = 84


def run(n, engines, steps, iterations, chain=False, graph=False):
    rng = np.random.default_rng(1)
    pool = Pool(tuple(ModelProfile(f"m{i}", 1.0 + i, 64) for i in range(engines)))
    cap = n
    gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(8, 4), router=ScoreTableRouter(),
                      predictor=PrecomputedPredictor(), n_programs=16, max_rows=16,
                      queue_capacity=cap)
    st = gs.state
    for m in range(engines):
        prio = np.maximum(1, np.round(rng.lognormal(np.log(650.0) - 0.5, 1.0, n)))
        arr = np.sort(rng.random(n) * 900.0)
        st.load_queue(m, prio, arr, np.arange(n), np.arange(n) + (m << 40),
                      level=-rng.integers(0, 2, n), count=rng.integers(0, 8, n))
    # engines full (work conservation: free slots imply an empty queue); each
    # tick 32 running requests complete, freeing slots the queue refills
    st.set_engine_counters(running=[64] * engines)
    n_complete = torch.full((engines,), 32, dtype=torch.int32, device=gs.device)
    gs.router.set(torch.zeros((0, engines), device=gs.device))
    gs.predictor.set(torch.zeros((0, engines), dtype=torch.float64, device=gs.device))
    empty = RowBatch.from_numpy(gs.device, program=np.zeros(0), stage=np.zeros(0),
                                arrival=np.zeros(0), out_tokens=np.zeros((0, engines)),
                                handle=np.zeros(0))
    snap = st.snapshot()
    for _ in range(2):
        st.restore(snap)
        gs.run_rows(empty, n_iterations=iterations, n_complete=n_complete)
    torch.cuda.synchronize()
    gs.check_errors()
    if graph:  # the tick as a CUDA-graph replay (how TickGraph runs it), CUDA events
        from paper_2603_22206_b200.tick import TickGraph
        st.restore(snap)
        tg = TickGraph(gs, empty, n_iterations=iterations, n_complete=n_complete,
                       restore_snapshot=None if chain else snap)
        for _ in range(2):
            tg.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            tg.replay()
        e1.record()
        torch.cuda.synchronize()
        gs.check_errors()
        ms = e0.elapsed_time(e1) / steps
        if not chain:  # the replay includes the snapshot restore: time it alone and subtract
            e0.record()
            for _ in range(steps):
                st.restore(snap)
            e1.record()
            torch.cuda.synchronize()
            ms -= e0.elapsed_time(e1) / steps
        calls = 2
    else:
        ms, calls = None, None
    _lib.profile_read()
    _lib.profile_enable(not graph)
    if graph:
        pass
    elif chain:  # one untimed tick so the timed ones continue a kept order
        st.restore(snap)
        gs.run_rows(empty, n_iterations=iterations, n_complete=n_complete)
        torch.cuda.synchronize()
        _lib.profile_read()
    for _ in range(0 if graph else steps):
        if not chain:
            st.restore(snap)
        gs.run_rows(empty, n_iterations=iterations, n_complete=n_complete)
    torch.cuda.synchronize()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    gs.check_errors()
    # two queue calls per tick: completions (admit into freed slots, age) and
    # the tick itself (append, iterate, final STJF order)
    if not graph:
        ms = prof["queue"]["ms"] / steps
        calls = prof["queue"]["timed"] / steps
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6549.1
    gbs = calls * n * engines * BYTES_PER_ENTRY / (ms / 1e3) / 1e9
    path = ("smem keys, 1 CTA/engine" if cap <= 10240 else
            "global keys, 1 CTA/engine" if cap <= (1 << 18) else "grid-wide passes")
    return {"entries_per_engine": n, "engines": engines, "capacity": cap, "path": path,
            "mode": ("chain (incremental)" if chain else "restored (radix)")
                    + (", graph replay" if graph else ", eager"),
            "iterations": iterations, "ms_per_tick": ms, "achieved_gbs": gbs,
            "peak_gbs": peak, "frac": gbs / peak,
            "bytes_per_entry": BYTES_PER_ENTRY}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[8192, 65536, 1 << 20, 1 << 24])
    ap.add_argument("--engines", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--iterations", type=int, default=1)
    ap.add_argument("--chain", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="time the tick as a CUDA-graph replay (whole tick: both queue calls)")
    a = ap.parse_args()
    for n in a.n:
        print(json.dumps(run(n, a.engines, a.steps, a.iterations, a.chain, a.graph)), flush=True)


if __name__ == "__main__":
    main()
