#!/usr/bin/env bash
# Flash v5 with two threads per query row (CHM_FLASH5_SPLIT=1, 16 softmax
# warps) vs one (0), polynomial share 2-5 of 8 exp2 pairs; parity of split.
cd "$(dirname "$0")/../.."
for sp in 0 1; do for p in 2 3 4 5; do
  echo -n "split $sp poly $p: "; CHM_FLASH5_SPLIT=$sp CHM_FLASH5_POLY=$p timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 10
done; done
CHM_FLASH5_SPLIT=1 timeout 300 python -m pytest tests -m gpu -q -k "attention_matches or long_prompts or random_layernorm" 2>&1 | tail -1
for m in 16 18 48; do echo "== split timeline mode $m"; CHM_FLASH5_SPLIT=1 CHM_FLASH5_ISSUE=$m timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --flash-timeline | tail -6; done
