#!/usr/bin/env bash
# Fused QKV+attention pair kernel: projection k-blocks kept queued ahead of
# S / O (CHM_QA_PAIR_LAG; 0 = the ring's depth). Kernel time at cfg3 shape
# (tools/attn_micro.py) and parity of the fused kernel at each lag.
cd "$(dirname "$0")/../.."
for lag in 0 1 2 3 4; do
  echo "== lag $lag"
  CHM_QA_PAIR_LAG=$lag python tools/attn_micro.py --only fused --reps 20
  CHM_QA_PAIR_LAG=$lag python -m pytest tests/test_gpu_attention.py -q -k "qkv_attention or fused_equals" 2>&1 | tail -1
done
for lag in 0 2; do
  echo "== timeline lag $lag"
  CHM_QA_DEBUG=11 CHM_QA_PAIR_LAG=$lag python tools/attn_micro.py --timeline
done
