"""Trace store micro-benchmark: chm_trace_derive HBM
throughput against the measured copy bandwidth, and the per-tick gathers
(oracle predictions + out_tokens for a 4096-row batch, next-stage requests for
a burst of completions), CUDA events, inputs resident in HBM. The CPU side is
the reference's own per-record accessors (TraceRecord.remaining_tokens /
next_stage_request semantics, restated in oracle/trace_ref.py as loops) on a
bounded sample.

  python tools/trace_bench.py [--programs 10000000] [--stages 8] [--models 5]
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
    ap.add_argument("--programs", type=int, default=10_000_000)
    ap.add_argument("--stages", type=int, default=8)
    ap.add_argument("--models", type=int, default=5)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    from paper_2603_22206_b200 import _lib
    from paper_2603_22206_b200.trace import TraceColumns, TraceStore

    NP, S, K = a.programs, a.stages, a.models
    rng = np.random.default_rng(1)
    c = TraceColumns(0, S, [f"m{k}" for k in range(K)])
    c.program_ids = [""] * NP
    c.workflow_ids = ["wf"] * NP
    c.n_stages = rng.integers(1, S + 1, NP).astype(np.int32)
    live = np.arange(S)[None, :] < c.n_stages[:, None]
    c.base_input = np.where(live, rng.integers(1, 4000, (NP, S)), 0).astype(np.int32)
    c.out_tokens = np.where(live[..., None], rng.integers(0, 4000, (NP, S, K)), 0).astype(np.int32)
    c.carried = c.out_tokens.copy()
    c.user_arrival = np.zeros(NP)
    st = TraceStore(c, "cuda")
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    lib = _lib.load()
    s = torch.cuda.current_stream()

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    ms_derive = timed(lambda: lib.chm_trace_derive(st.t, st.error.data_ptr(), s.cuda_stream),
                      a.reps)
    gbs = st.bytes_derive / (ms_derive * 1e-3) / 1e9
    B = 4096
    prog = torch.randint(0, NP, (B,), dtype=torch.int32, device="cuda")
    stage = torch.ones(B, dtype=torch.int32, device="cuda")
    yhat = torch.empty(B, K, dtype=torch.float64, device="cuda")
    outt = torch.empty(B, K, dtype=torch.int32, device="cuda")
    ms_gather = timed(lambda: lib.chm_trace_gather_rows(
        st.t, prog.data_ptr(), stage.data_ptr(), B, outt.data_ptr(), None, None,
        yhat.data_ptr(), st.error.data_ptr(), s.cuda_stream), a.reps * 10)
    NC = 65536
    cp = torch.randint(0, NP, (NC,), dtype=torch.int32, device="cuda")
    cs = torch.ones(NC, dtype=torch.int32, device="cuda")
    ct = torch.zeros(NC, dtype=torch.float64, device="cuda")
    cm = torch.randint(0, K, (NC,), dtype=torch.int8, device="cuda")
    bufs = [torch.empty(NC, dtype=dt, device="cuda") for dt in
            (torch.int32, torch.int32, torch.float64, torch.int32)]
    nn = torch.zeros(1, dtype=torch.int32, device="cuda")
    ms_next = timed(lambda: lib.chm_trace_next_stage(
        st.t, cp.data_ptr(), cs.data_ptr(), ct.data_ptr(), cm.data_ptr(), NC,
        *(b.data_ptr() for b in bufs), None, None, nn.data_ptr(), st.error.data_ptr(),
        s.cuda_stream), a.reps * 10)
    st.check_errors("bench")
    # CPU: per-record accessors, as the reference answers them (loops over
    # stages per (program, model) call), on a bounded sample of programs
    n_cpu = 20000
    o = c.out_tokens[:n_cpu].tolist()
    ns = c.n_stages[:n_cpu].tolist()
    t0 = time.perf_counter()
    for p in range(n_cpu):
        for s_ in range(1, ns[p] + 1):
            for k in range(K):
                sum(o[p][j][k] for j in range(s_ - 1, ns[p]))
    cpu_s = time.perf_counter() - t0
    entries = int(np.sum(c.n_stages[:n_cpu])) * K
    print(json.dumps({
        "kernel": "chm::trace::derive_kernel", "programs": NP, "stages": S, "models": K,
        "derive_ms": ms_derive, "derive_bytes": st.bytes_derive, "derive_GBps": gbs,
        "hbm_peak_GBps": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
        "gather_4096_rows_us": ms_gather * 1e3, "next_stage_65536_us": ms_next * 1e3,
        "cpu_remaining_entries_per_s": entries / cpu_s,
        "gpu_remaining_entries_per_s": NP * S * K / (ms_derive * 1e-3),
        "cpu_sample": f"{n_cpu} programs, remaining_tokens for every (stage, model), 1 thread",
    }))


if __name__ == "__main__":
    main()
