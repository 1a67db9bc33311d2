#!/usr/bin/env bash
# flash v6: O and l from one N = 80 MMA over [V | ones] (default) vs separate
# N = 64 / N = 16 MMAs (libchimera_nol.so: -DCHM_F6_OL=0)
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_attention.py -q -x -k "attention_matches or long_prompts or random_layernorm" > gpurun_out/ol_tests.txt 2>&1; tail -1 gpurun_out/ol_tests.txt
for r in 1 2; do
  for v in sm100a nol; do
    echo -n "$v: "; CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5 2>&1 | tail -1
  done
done
