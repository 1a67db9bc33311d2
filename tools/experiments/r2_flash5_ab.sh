#!/usr/bin/env bash
# flash v5 on one box: CHM_FLASH5_POLY = exp2 pairs (of 8) computed by the
# FMA-pipe polynomial instead of MUFU. Alternated, 2 rounds, then parity.
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for d in ${POLYS:-0 1 2 3}; do
    echo -n "poly=$d "
    CHM_FLASH=5 CHM_FLASH5_POLY=$d timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
  done
done
for d in ${POLYS:-0 1 2 3}; do
  CHM_FLASH=5 CHM_FLASH5_POLY=$d timeout 300 python -m pytest tests -m gpu -q -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -1
done
