#!/usr/bin/env bash
# Fused QKV+attention pair kernel: the two CTAs' S / O MMAs issued together
# (CHM_QA_PAIR_SYNC=1) or independently (0).
cd "$(dirname "$0")/../.."
for v in 0 1; do
  echo "== CHM_QA_PAIR_SYNC=$v"
  for r in 1 2; do CHM_QA_PAIR_SYNC=$v timeout 120 python tools/attn_micro.py --only fused --reps 20; done
  CHM_QA_PAIR_SYNC=$v timeout 300 python -m pytest tests/test_gpu_attention.py -q -k "qkv_attention or fused_equals" 2>&1 | tail -1
  CHM_QA_PAIR_SYNC=$v CHM_QA_DEBUG=11 timeout 120 python tools/attn_micro.py --timeline | tail -4
done
