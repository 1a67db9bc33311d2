#!/usr/bin/env bash
# Flash v5: MMA pipeline alone (mode|32: softmax skipped), softmax alone
# (mode|64: no MMAs), both; per-block timelines (|16) and kernel times.
cd "$(dirname "$0")/../.."
for m in 0 2 32 34 64 66; do
  echo "== mode $m"; CHM_FLASH5_ISSUE=$m timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 10
done
for m in 48 50 80 82; do echo "== timeline mode $m"; CHM_FLASH5_ISSUE=$m timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --flash-timeline | tail -12; done
