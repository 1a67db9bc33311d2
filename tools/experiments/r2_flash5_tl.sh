#!/usr/bin/env bash
# Flash v5 per-block timeline of CTA 0 (issue modes 0 / 1 / 2 | 16)
cd "$(dirname "$0")/../.."
for m in 16 17 18; do echo "== mode $m"; CHM_FLASH5_ISSUE=$m timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --flash-timeline; done
