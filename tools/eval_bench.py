"""Kendall-tau distance on the device vs the reference's pure-Python
algorithm (oracle/eval_ref.py restates it) -- SURVEY §8f row 4.

  python tools/eval_bench.py [--n 16777216]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from oracle import eval_ref
    from paper_2603_22206_b200 import _lib
    from paper_2603_22206_b200.evaluate import kendall_tau_distance

    g = torch.Generator(device="cuda").manual_seed(1)
    p = torch.randint(0, 4000, (a.n,), device="cuda", generator=g).double()
    t = torch.randint(0, 4000, (a.n,), device="cuda", generator=g).double()
    kendall_tau_distance(p, t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        d = kendall_tau_distance(p, t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    n_cpu = 200_000
    pc, tc = p[:n_cpu].cpu().tolist(), t[:n_cpu].cpu().tolist()
    t0 = time.perf_counter()
    eval_ref.ref_kendall_counts(pc, tc)
    cpu_s = time.perf_counter() - t0
    print(json.dumps({"n": a.n, "gpu_ms": ms, "gpu_pairs_per_s": a.n / (ms * 1e-3),
                      "distance": d, "cpu_sample": n_cpu, "cpu_s": cpu_s,
                      "cpu_pairs_per_s": n_cpu / cpu_s,
                      "note": "GPU time includes the scratch allocation and result read-back"}))


if __name__ == "__main__":
    main()
