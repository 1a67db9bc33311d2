#!/usr/bin/env bash
# duo fused kernel: W slices multicast across two pairs (CHM_QA_DUO_MC=1) vs not
cd "$(dirname "$0")/../.."
CHM_QA_DUO_MC=1 timeout 120 python -m pytest tests/test_gpu_attention.py -q -x -k "qkv_attention or fused" 2>&1 | tail -2
for r in 1 2; do for H in 768 256; do for m in 0 1; do
  echo -n "H $H mc $m: "; CHM_QA_DUO_MC=$m timeout 60 python tools/attn_micro.py --hidden $H --only fused --reps 20
done; done; done
