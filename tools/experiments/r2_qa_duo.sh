#!/usr/bin/env bash
# fused QKV+attention: two-epilogue-group kernel (CHM_QA_DUO=1, default) vs the
# PAIR kernel (0): parity and kernel time at H = 768 / 256
cd "$(dirname "$0")/../.."
timeout 120 python -m pytest tests/test_gpu_attention.py -q -x -k "qkv_attention" 2>&1 | tail -3
for H in 768 256; do for d in 1 0; do
  echo -n "H $H duo $d: "; CHM_QA_DUO=$d timeout 60 python tools/attn_micro.py --hidden $H --only fused --reps 20
done; done
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_router.py tests/test_gpu_tick.py -q -x 2>&1 | tail -2
