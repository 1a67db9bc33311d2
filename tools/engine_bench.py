"""Engine-side micro-benchmarks for SURVEY §8f rows 1 and 3 (CUDA events,
state resident in HBM):

* engine clock: K engines with Q queued requests each and b slots;
  chm_engine_advance over successive windows, each finishing ~`--per-window`
  stints per engine. Every finish runs a scheduling iteration (admit +
  aging). Reported as stint completions per second.
* global admission: one sharded scheduling iteration per engine
  (chm_queue_candidates + chm_queue_admit_merged) with G simulated ranks'
  candidates, timed without the all-gather (which is NCCL's).

  python tools/engine_bench.py [--models 8] [--queued 8192] [--batch 32]
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", type=int, default=8)
    ap.add_argument("--queued", type=int, default=8192)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--per-window", type=int, default=256)
    ap.add_argument("--windows", type=int, default=20)
    ap.add_argument("--ranks", type=int, default=8)
    a = ap.parse_args()
    from paper_2603_22206_b200.config import AgingConfig, ModelProfile, Pool
    from paper_2603_22206_b200.predictor import PrecomputedPredictor
    from paper_2603_22206_b200.router import ScoreTableRouter
    from paper_2603_22206_b200.scheduler import GpuScheduler

    K, Qn, b = a.models, a.queued, a.batch
    rng = np.random.default_rng(7)
    d_ms = [0.5 + 0.5 * k for k in range(K)]
    pool = Pool(tuple(ModelProfile(f"m{k}", d_ms[k], b, prefill_ms_per_token=0.02)
                      for k in range(K)))
    out = {}

    def fresh(engine_clock):
        rt, pr = ScoreTableRouter(), PrecomputedPredictor()
        rt.set(torch.zeros((0, K), dtype=torch.float32, device="cuda"))
        pr.set(torch.zeros((0, K), dtype=torch.float64, device="cuda"))
        gs = GpuScheduler(pool, aging=AgingConfig(starvation_threshold=8),
                          router=rt, predictor=pr,
                          n_programs=8, max_rows=8, queue_capacity=Qn + 1024,
                          engine_clock=engine_clock, completion_capacity=Qn + 2 * b)
        st = gs.state
        for m in range(K):
            st.load_queue(m, rng.integers(1, 4000, Qn).astype(np.float64), np.zeros(Qn),
                          np.arange(Qn), m * 10 ** 6 + np.arange(Qn),
                          out_tokens=rng.integers(16, 600, Qn))
            st.engine_seq[m] = Qn
        if engine_clock:
            st.q_input_tokens.copy_(torch.as_tensor(
                rng.integers(64, 2048, K * (Qn + 1024)), dtype=torch.int32))
        return gs

    # ---- engine clock -----------------------------------------------------
    gs = fresh(True)
    gs.scheduling_iteration(1)  # fill the running batches at t = 0
    gs.check_errors()
    # window length: per-window stints at the mean stint time / b slots
    mean_stint = 0.02 * 1056 + np.mean(d_ms) * 308
    dt = a.per_window * mean_stint / b
    t = 0.0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):  # warm-up windows
        t += dt
        gs.advance_to(t)
    torch.cuda.synchronize()
    n_done = 0
    ev0.record()
    for _ in range(a.windows):
        t += dt
        gs.advance_to(t, keep_completions=True)
    ev1.record()
    torch.cuda.synchronize()
    gs.check_errors()
    n_done = int(gs.state.run_n_done.sum())
    ms = ev0.elapsed_time(ev1)
    out["engine_clock"] = dict(
        kernel="chm::queue_kernel mode 3 (chm_engine_advance)", engines=K, queued=Qn, batch=b,
        windows=a.windows, completions=n_done, ms=ms,
        completions_per_s=n_done / (ms / 1e3), us_per_window=ms * 1e3 / a.windows,
        iterations=int(gs.state.engine_iterations.sum()))

    # ---- global admission (one merged iteration) ---------------------------
    gs = fresh(False)
    st = gs.state
    gs.scheduling_iteration(0)  # STJF order of the loaded queues
    cand = gs.queue_candidates()
    G = a.ranks
    gathered = torch.stack([cand] * G).clone()
    gathered[1:, :, :, 3] += 1 << 40  # other ranks' entries: later seq, distinct keys
    snap = {k: v.clone() for k, v in st.snapshot().items()}
    for _ in range(3):
        st.restore(snap)
        gs.queue_admit_merged(gathered, 0)
    torch.cuda.synchronize()
    reps = 20
    tot = 0.0
    for _ in range(reps):
        st.restore(snap)
        ev0.record()
        c = gs.queue_candidates()
        gs.queue_admit_merged(gathered, 0)
        ev1.record()
        torch.cuda.synchronize()
        tot += ev0.elapsed_time(ev1)
    gs.check_errors()
    del c
    out["global_admission"] = dict(
        kernels="chm_queue_candidates + chm_queue_admit_merged", engines=K, queued=Qn,
        ranks=G, candidates_per_rank=b, us_per_iteration=tot * 1e3 / reps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
