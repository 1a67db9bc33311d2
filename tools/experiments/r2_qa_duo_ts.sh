#!/usr/bin/env bash
# duo fused kernel: Q / P in TMEM (CHM_QA_DUO_TS=1) vs shared memory (0)
cd "$(dirname "$0")/../.."
CHM_QA_DUO_TS=1 timeout 120 python -m pytest tests/test_gpu_attention.py -q -x -k "qkv_attention or fused" 2>&1 | tail -1
for r in 1 2; do for H in 768 256; do for t in 0 1; do
  echo -n "H $H ts $t: "; CHM_QA_DUO_TS=$t timeout 60 python tools/attn_micro.py --hidden $H --only fused --reps 20
done; done; done
