"""Micro-benchmark of the router's four GEMM shapes at the cfg3 token count
(M = 4096 x 128), CUDA events, inputs resident in HBM.

  python tools/gemm_micro.py [--m 524288] [--reps 10]
"""

import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_22206_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096 * 128)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    lib = _lib.load()
    M, H, F = a.m, 768, 3072
    dev = "cuda"
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn(M, H, device=dev).to(torch.bfloat16)
    f = torch.randn(M, F, device=dev).to(torch.bfloat16)
    out_h = torch.empty(M, H, dtype=torch.bfloat16, device=dev)
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
    }
    for name, (fn, fl) in cases.items():
        if a.only and a.only not in name:
            continue
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{name:10s} {ms:8.3f} ms  {fl / ms / 1e9:8.1f} TFLOP/s")


if __name__ == "__main__":
    main()
