#!/usr/bin/env bash
# K7 radix pass with per-warp slices (one scan per pass): parity + cfg4/cfg1/cfg3 ticks
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x -k "queue or engine_clock or complete or tick or schedule or shard or evaluate or bench" 2>&1 | tail -2
for c in cfg4 cfg1 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/rp_$c.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/rp_$c.json').read().strip().splitlines()[-1]);print('$c', round(d['ms_per_step'],3), round(d['value']), 'queue', round(d['stages_ms_per_tick']['queue'],3))"
done
