#!/usr/bin/env bash
# Fused QKV+attention pair kernel with a 5- (default) vs 6-stage operand ring
# (libchimera_qa6.so: -DCHM_QA_PAIR_STAGES=6, 223 KB of shared memory).
cd "$(dirname "$0")/../.."
for lib in libchimera_sm100a.so libchimera_qa6.so; do
  echo "== $lib"
  for r in 1 2; do CHM_LIB=paper_2603_22206_b200/$lib python tools/attn_micro.py --only fused --reps 20; done
  CHM_LIB=paper_2603_22206_b200/$lib python -m pytest tests/test_gpu_attention.py -q -k "qkv_attention or fused_equals" 2>&1 | tail -1
  CHM_LIB=paper_2603_22206_b200/$lib CHM_QA_DEBUG=11 python tools/attn_micro.py --timeline | tail -4
done
