#!/usr/bin/env bash
# flash v7 (P in its own TMEM columns, S(j+1) issued once S(j) is in registers)
# (v7 was removed after this measurement -- see profiles/r2_flash5_analysis.md;
# CHM_FLASH=7 no longer selects it)
# vs v6 / v5 on one box, then v7 parity and CTA 0's per-block stamps.
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for v in 5 6 7; do
    echo -n "flash v$v "
    CHM_FLASH=$v timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
  done
done
for p in ${POLYS:-2 4}; do
  echo -n "flash v7 poly $p "
  CHM_FLASH=7 CHM_FLASH6_POLY=$p timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
done
CHM_FLASH=7 timeout 300 python -m pytest tests -m gpu -q -x -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -3
CHM_FLASH=7 CHM_FLASH5_ISSUE=16 timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 1 --flash-timeline 2>&1 | tail -8
