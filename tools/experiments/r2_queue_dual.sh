#!/usr/bin/env bash
# K7 dual layout (shared-memory keys when a big-capacity segment holds <= 10240 entries)
# (the dual-layout kernel was measured from a working tree -- slower, 0.498 vs
# 0.469 ms at cfg4 -- and not committed; CHM_QUEUE_DUAL no longer exists)
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x -k "queue or engine_clock or complete or tick or bench" 2>&1 | tail -2
for r in 1 2; do
  for v in 1 0; do
    CHM_QUEUE_DUAL=$v timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/q_$v.json 2>/dev/null
    python -c "
import json;d=json.loads(open('gpurun_out/q_$v.json').read().strip().splitlines()[-1]);print('dual=$v', round(d['ms_per_step'],3), round(d['value']), 'queue', round(d['stages_ms_per_tick']['queue'],3))"
  done
done
