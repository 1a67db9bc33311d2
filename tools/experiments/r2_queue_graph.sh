#!/usr/bin/env bash
# K7 16.8M-entry tick: eager vs CUDA-graph replay, restored vs chained
cd "$(dirname "$0")/../.."
for m in "" "--chain"; do for g in "" "--graph"; do
  timeout 600 python tools/queue_stress.py --n 16777216 --steps 5 $m $g
done; done
