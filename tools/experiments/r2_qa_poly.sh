#!/usr/bin/env bash
# Fused QKV+attention (cfg3 shape): softmax exp2 pairs (of 4) on the FMA pipes,
# CHM_QA_POLY = 0 (default build) / 1 / 2 (tools/build_variant.py builds).
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for lib in libchimera_sm100a.so libchimera_qapoly1.so libchimera_qapoly2.so; do
    echo -n "$lib "
    CHM_LIB=paper_2603_22206_b200/$lib python tools/attn_micro.py --only fused --reps 20 | tail -1
  done
done
for lib in libchimera_sm100a.so libchimera_qapoly1.so libchimera_qapoly2.so; do
  CHM_LIB=paper_2603_22206_b200/$lib python -m pytest tests/test_gpu_attention.py -q -k "qkv_attention or fused_equals" 2>&1 | tail -1
done
