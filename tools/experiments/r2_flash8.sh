#!/usr/bin/env bash
# flash v8 (v6 with two threads per query row) vs v6; parity; stamps
# (the v8 kernel was measured from a working tree and not committed; this
# script records the commands; CHM_FLASH=8 no longer selects it)
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for v in 6 8; do
    echo -n "flash v$v "
    CHM_FLASH=$v timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
  done
done
for p in ${POLYS:-2 4}; do
  echo -n "flash v8 poly $p "
  CHM_FLASH=8 CHM_FLASH6_POLY=$p timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 5
done
CHM_FLASH=8 timeout 300 python -m pytest tests -m gpu -q -x -k "attention_matches or long_prompts or random_layernorm or cls_pool" 2>&1 | tail -2
CHM_FLASH=8 CHM_FLASH5_ISSUE=16 timeout 120 python tools/attn_micro.py --seq-len 512 --n-seq 2048 --only attention --reps 1 --flash-timeline 2>&1 | tail -3
