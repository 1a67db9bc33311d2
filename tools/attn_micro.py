"""Micro-benchmark of the S = 128 attention sublayer core at the cfg3 shape:
fused QKV+attention kernel vs QKV GEMM + attention kernel (CUDA events).

  python tools/attn_micro.py [--n-seq 4096] [--hidden 768] [--reps 10] [--only fused|unfused]
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
    ap.add_argument("--n-seq", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=768)
    ap.add_argument("--seq-len", type=int, default=128)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    ap.add_argument("--timeline", action="store_true",
                    help="with CHM_QA_DEBUG=11: print CTA 0's per-item stage stamps (cycles)")
    ap.add_argument("--flash-timeline", action="store_true",
                    help="with CHM_FLASH5_ISSUE |= 16: CTA 0's per-block flash v5 stamps (cycles)")
    a = ap.parse_args()
    lib = _lib.load()
    n, H, S = a.n_seq, a.hidden, a.seq_len
    T = n * S
    dev = "cuda"
    x = torch.randn(T, H, device=dev).to(torch.bfloat16)
    w = (torch.randn(3 * H, H, device=dev) / math.sqrt(H)).to(torch.bfloat16)
    b = torch.randn(3 * H, device=dev) * 0.1
    qkv = torch.empty(T, 3 * H, dtype=torch.bfloat16, device=dev)
    ctx = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
    st = torch.cuda.current_stream().cuda_stream

    def fused():
        _lib.check(lib.chm_qkv_attention_bf16(x.data_ptr(), w.data_ptr(), b.data_ptr(),
                                              ctx.data_ptr(), n, H, st), "fused")

    def gemm():
        _lib.check(lib.chm_gemm_bf16(x.data_ptr(), w.data_ptr(), qkv.data_ptr(), b.data_ptr(),
                                     None, T, 3 * H, H, 1, st), "gemm")

    def attn():
        _lib.check(lib.chm_attention_bf16(qkv.data_ptr(), ctx.data_ptr(), n, S, H, st), "attn")

    flops_g = 2.0 * T * 3 * H * H
    flops_a = 4.0 * S * S * 64 * n * (H // 64)
    cases = {"fused": (fused, flops_g + flops_a), "gemm": (gemm, flops_g),
             "attention": (attn, flops_a)}
    if os.environ.get("CHM_QA_DUO_TL"):
        fused()
        torch.cuda.synchronize()
        t = ctx.view(-1).view(torch.int64)[:32 * 12].cpu().view(32, 12).numpy()
        base = int(t[8, 0])
        names = ["acc_full", "staged", "s_full", "p_ready", "o_full", "out", "S_iss", "O_iss",
                 "buf_free", "kb0", "kbN"]
        print("item " + " ".join(f"{n:>8s}" for n in names) + "   (cycles from item 8 acc_full)")
        for i in range(8, 20):
            print(f"{i:4d} " + " ".join(f"{int(v) - base:8d}" for v in t[i][:11]))
        return
    if a.flash_timeline and os.environ.get("CHM_FLASH") in ("6", "7"):
        attn()
        torch.cuda.synchronize()
        t = ctx.view(-1).view(torch.int64)[:256].cpu().view(64, 4).numpy()
        base = int(t[4, 0])
        names = ["S0_land", "P0_done", "S1_land", "P1_done"]
        print("blk " + " ".join(f"{n:>9s}" for n in names) + "   (cycles from block 4 S0_land)")
        for j in range(4, 24):
            print(f"{j:3d} " + " ".join(f"{int(v) - base:9d}" for v in t[j]))
        d = t[8:40]
        per = (int(d[-1, 1]) - int(d[0, 1])) / (len(d) - 1)
        print(f"period {per:.0f} cycles per 128-key block; softmax S->P tile0 "
              f"{float((d[:,1]-d[:,0]).mean()):.0f}, tile1 {float((d[:,3]-d[:,2]).mean()):.0f}; "
              f"P0(j)->S0(j+1) {float((d[1:,0]-d[:-1,1]).mean()):.0f}; "
              f"S0->S1 land offset {float((d[:,2]-d[:,0]).mean()):.0f}")
        return
    if a.flash_timeline:
        attn()
        torch.cuda.synchronize()
        t = ctx.view(-1).view(torch.int64)[:512].cpu().view(64, 8).numpy()
        base = int(t[8, 0])
        names = ["S0_land", "P0_done", "S1_land", "P1_done", "O0_iss", "S0+2_iss", "O1_iss", "S1+2_iss"]
        print("blk " + " ".join(f"{n:>9s}" for n in names) + "   (cycles from block 8 S0_land)")
        for j in range(8, 40):
            print(f"{j:3d} " + " ".join(f"{int(v) - base:9d}" for v in t[j]))
        d = t[16:48]
        per = (int(d[-1, 1]) - int(d[0, 1])) / (len(d) - 1)
        print(f"period {per:.0f} cycles/block; softmax S->P tile0 {float((d[:,1]-d[:,0]).mean()):.0f}, "
              f"tile1 {float((d[:,3]-d[:,2]).mean()):.0f}; P0->S0(j+1) land wait "
              f"{float((d[1:,0]-d[:-1,1]).mean()):.0f}")
        return
    if a.timeline:
        fused()
        torch.cuda.synchronize()
        t = ctx.view(-1).view(torch.int64)[:128].cpu().view(8, 16)[:, :13]
        base = int(t[0, 0])
        names = ["acc_full", "staged", "s_full", "p_ready", "o_full", "out_done", "S_issue", "O_issue",
                 "acc_free", "kb0_mma", "kbN_mma", "kb0_tma", "kbN_tma"]
        print("item " + " ".join(f"{n:>8s}" for n in names) + "   (cycles from item 8 acc_full)")
        for i in range(8):
            print(f"{8 + i:4d} " + " ".join(f"{int(v) - base:8d}" for v in t[i]))
        return
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
