"""Micro-benchmark of the router's four GEMM shapes at the cfg3 token count
(M = 4096 x 128), CUDA events, inputs resident in HBM.

  python tools/gemm_micro.py [--m 524288] [--reps 10]
"""

import argparse
import math
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_22206_b200 import _lib  # noqa: E402


class ClockProbe:
    """Median SM clock (NVML) sampled every 2 ms while a case runs."""

    def __init__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        except Exception:  # noqa: BLE001
            self.nv = None

    def start(self):
        import threading
        self.samples, self.run = [], True
        def loop():
            while self.run:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                time.sleep(0.002)
        if self.nv:
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()

    def energy_mj(self):
        return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) if self.nv else 0

    def stop(self):
        if not self.nv:
            return 0.0
        self.run = False
        self.t.join()
        s = sorted(self.samples)
        return float(s[len(s) // 2]) if s else 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096 * 128)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--seconds", type=float, default=0.0,
                    help="> 0: repeat each case for about this long (energy per launch from NVML)")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    lib = _lib.load()
    M, H, F = a.m, 768, 3072
    dev = "cuda"
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn(M, H, device=dev).to(torch.bfloat16)
    f = torch.randn(M, F, device=dev).to(torch.bfloat16)
    out_h = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
    x2 = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
    out_q = torch.empty(M, 3 * H, dtype=torch.bfloat16, device=dev)
    out_f = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
    w = {n: (torch.randn(r, c, device=dev) / math.sqrt(c)).to(torch.bfloat16)
         for n, (r, c) in {"qkv": (3 * H, H), "o": (H, H), "1": (F, H), "2": (H, F)}.items()}
    b = torch.randn(F * 3, device=dev) * 0.1
    g = torch.ones(H, device=dev)
    be = torch.zeros(H, device=dev)

    def plain(A, W, C, N, K, epi):
        return lambda: _lib.check(lib.chm_gemm_bf16(A.data_ptr(), W.data_ptr(), C.data_ptr(),
                                                    b.data_ptr(), None, M, N, K, epi, st), "g")

    def ln(A, W, C, K):
        return lambda: _lib.check(lib.chm_gemm_bf16_ln(A.data_ptr(), W.data_ptr(), C.data_ptr(),
                                                       b.data_ptr(), x.data_ptr(), g.data_ptr(),
                                                       be.data_ptr(), 1e-12, M, H, K, st), "ln")

    P = H // 128
    st_a = torch.zeros(M, P, 2, device=dev)
    st_a[..., 1] = 127.0
    st_b = torch.empty(M, P, 2, device=dev)
    csum = torch.randn(F, device=dev)

    def deferred(A, W, C, N, K, epi, res=None, stats_in=None, stats_out=None):
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        return lambda: _lib.check(lib.chm_gemm_bf16_deferred_ln(
            A.data_ptr(), W.data_ptr(), C.data_ptr(), b.data_ptr(), epi, ptr(res), g.data_ptr(),
            be.data_ptr(), ptr(stats_in), P, csum.data_ptr(), ptr(stats_out), 1e-12, M, N, K,
            st), "d")

    def cublas(A, W, C):
        return lambda: torch.matmul(A, W.t(), out=C)

    cases = {
        "cublas_qkv": (cublas(x, w["qkv"], out_q), 2.0 * M * 3 * H * H),
        "cublas_ffn1": (cublas(x, w["1"], out_f), 2.0 * M * F * H),
        "cublas_ffn2": (cublas(f, w["2"], out_h), 2.0 * M * H * F),
        "qkv": (plain(x, w["qkv"], out_q, 3 * H, H, 1), 2.0 * M * 3 * H * H),
        "out_ln": (ln(out_h, w["o"], out_h, H), 2.0 * M * H * H),
        "ffn1_gelu": (plain(x, w["1"], out_f, F, H, 2), 2.0 * M * F * H),
        "ffn2_ln": (ln(f, w["2"], out_h, F), 2.0 * M * H * F),
        "out_resln": (deferred(out_h, w["o"], x2, H, H, 6, x, st_a, st_b), 2.0 * M * H * H),
        "ffn1_fold": (deferred(x, w["1"], out_f, F, H, 2, None, st_a), 2.0 * M * F * H),
        "ffn2_resln": (deferred(f, w["2"], x2, H, F, 6, x, st_a, st_b), 2.0 * M * H * F),
    }
    clk = ClockProbe()
    for name, (fn, fl) in cases.items():
        if a.only and not any(o in name for o in a.only.split(",")):
            continue
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        reps = a.reps
        if a.seconds > 0:
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            reps = max(a.reps, int(a.seconds / max(time.perf_counter() - t0, 1e-6)))
        a_reps, a.reps = a.reps, reps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk.start()
        mj0 = clk.energy_mj()
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        mhz = clk.stop()
        joules = (clk.energy_mj() - mj0) * 1e-3 / reps
        ms = e0.elapsed_time(e1) / a.reps
        a.reps = a_reps
        # per-clock efficiency: FLOPs / (cycles x 148 SMs x 8192 dense bf16 FLOP/clk/SM)
        eff = fl / (ms * 1e-3 * mhz * 1e6 * 148 * 8192) if mhz else float("nan")
        print(f"{name:10s} {ms:8.3f} ms  {fl / ms / 1e9:8.1f} TFLOP/s  sm {mhz:6.0f} MHz  "
              f"tensor-eff {eff:5.3f}  {joules / (fl * 1e-12):6.3f} J/TFLOP  "
              f"{joules / (ms * 1e-3):6.0f} W")


if __name__ == "__main__":
    main()
