#!/usr/bin/env bash
# flash v7 with the issuer in event order vs v6; parity; stamps
# (v7 was removed after this measurement -- see profiles/r2_flash5_analysis.md;
# CHM_FLASH=7 no longer selects it)
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for v in 6 7; do
    echo -n "flash v$v "
    CHM_FLASH=$v timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
  done
done
for p in ${POLYS:-2 1}; do
  echo -n "flash v7 poly $p "
  CHM_FLASH=7 CHM_FLASH6_POLY=$p timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
done
CHM_FLASH=7 timeout 300 python -m pytest tests -m gpu -q -x -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -3
CHM_FLASH=7 CHM_FLASH5_ISSUE=16 timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 1 --flash-timeline 2>&1 | tail -8
