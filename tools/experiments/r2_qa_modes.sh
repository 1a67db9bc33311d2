#!/usr/bin/env bash
# fused QKV+attention (PAIR): full kernel vs projection only (dbg 1), + Q/K/V
# staging (dbg 2); cfg3 shape (H 768) and the small router (H 256)
cd "$(dirname "$0")/../.."
for H in 768 256; do for d in 0 1 2; do
  echo -n "H $H dbg $d: "; CHM_QA_DEBUG=$d timeout 120 python tools/attn_micro.py --hidden $H --only fused --reps 20
done; done
for H in 256; do echo -n "H $H unfused: "; timeout 120 python tools/attn_micro.py --hidden $H --only gemm --reps 20; timeout 120 python tools/attn_micro.py --hidden $H --only attention --reps 20; done
