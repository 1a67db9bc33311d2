#!/usr/bin/env bash
# Flash attention (S = 512) v1 (round-1 softmax) vs v2 (thresholded rescale,
# P.ones row sums, partial polynomial exp2): kernel time at the cfg5 shape and
# parity of the long-prompt paths.
cd "$(dirname "$0")/../.."
for v in 0 1; do
  echo "== CHM_FLASH_V2=$v"
  CHM_FLASH_V2=$v python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
  CHM_FLASH_V2=$v python -m pytest tests -m gpu -q -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -1
done
