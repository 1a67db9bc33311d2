#!/usr/bin/env bash
# Flash attention (S = 512) versions: 1 round-1 kernel, 2 v2 softmax (P.ones
# row sums, thresholded rescale, partial polynomial exp2), 3 64-key blocks with
# double-buffered S and O resident in TMEM, 4 P in TMEM over S (TS MMAs), 5 64-key
# blocks with Q, P in TMEM and S issued two blocks ahead. Kernel time at the cfg5 shape and
# parity of the long-prompt paths.
cd "$(dirname "$0")/../.."
for v in ${FLASH_VERSIONS:-2 4 5}; do
  echo "== CHM_FLASH=$v"
  CHM_FLASH=$v timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
  CHM_FLASH=$v timeout 300 python -m pytest tests -m gpu -q -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -1
done
