#!/usr/bin/env bash
# Flash v5 MMA issue order: CHM_FLASH5_ISSUE 0 (S_g(j) waits for O_g(j-2) to
# complete; O0 O1 S0 S1), 1 (no wait, O0 S0 O1 S1), 2 (no wait, O0 O1 S0 S1).
cd "$(dirname "$0")/../.."
for m in ${MODES:-0 1 2}; do
  echo "== CHM_FLASH5_ISSUE=$m"
  for r in 1 2; do CHM_FLASH5_ISSUE=$m timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 10; done
  CHM_FLASH5_ISSUE=$m timeout 300 python -m pytest tests -m gpu -q -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -1
done
