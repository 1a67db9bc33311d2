"""Micro-benchmark: fused H = 256 FFN sublayer vs FFN1 (GELU) + FFN2 (LN) GEMMs
(CUDA events). python tools/ffn_micro.py [--m 524288] [--f 1024] [--reps 20]"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_22206_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=524288)
    ap.add_argument("--f", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lib = _lib.load()
    M, H, Fd = a.m, 256, a.f
    x = torch.randn(M, H, device="cuda").to(torch.bfloat16)
    w1 = (torch.randn(Fd, H, device="cuda") / math.sqrt(H)).to(torch.bfloat16)
    w2 = (torch.randn(H, Fd, device="cuda") / math.sqrt(Fd)).to(torch.bfloat16)
    b1 = torch.zeros(Fd, device="cuda")
    b2 = torch.zeros(H, device="cuda")
    g = torch.ones(H, device="cuda")
    hbuf = torch.empty(M, Fd, dtype=torch.bfloat16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream

    def fused():
        _lib.check(lib.chm_ffn_fused_bf16(x.data_ptr(), w1.data_ptr(), b1.data_ptr(),
                                          w2.data_ptr(), b2.data_ptr(), g.data_ptr(),
                                          b2.data_ptr(), 1e-12, M, H, Fd, st), "fused")

    def ffn1():
        _lib.check(lib.chm_gemm_bf16(x.data_ptr(), w1.data_ptr(), hbuf.data_ptr(), b1.data_ptr(),
                                     None, M, Fd, H, 2, st), "ffn1")

    def ffn2():
        _lib.check(lib.chm_gemm_bf16_ln(hbuf.data_ptr(), w2.data_ptr(), x.data_ptr(),
                                        b2.data_ptr(), x.data_ptr(), g.data_ptr(), b2.data_ptr(),
                                        1e-12, M, H, Fd, st), "ffn2")

    if int(os.environ.get("CHM_FFN_TL", "0")) & 1:
        fused()
        torch.cuda.synchronize()
        t = x.view(-1).view(torch.int64)[:48 * 8].cpu().view(48, 8).numpy()
        base = int(t[0, 0])
        print("chunk  acc_rdy  released  H_free  E1_done  G1_iss  G2_iss")
        for i in range(24):
            print(f"{i:5d} " + " ".join(f"{int(v) - base:8d}" for v in t[i][:6]))
        for i in range(32, 35):
            print(f"tile {i - 32}: Y ready {int(t[i][0]) - base}, done {int(t[i][1]) - base}")
        return
    flops = 4.0 * M * H * Fd
    for name, fn in (("fused", fused), ("ffn1", ffn1), ("ffn2", ffn2)):
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
        print(f"{name:6s} {ms:7.3f} ms  {(flops if name == 'fused' else flops / 2) / ms / 1e9:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
