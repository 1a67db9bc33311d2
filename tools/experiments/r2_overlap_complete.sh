#!/usr/bin/env bash
# completions on a side stream under the router (run_rows): parity, cfg4 tick
# (measured and reverted: no gain -- the 8 one-CTA-per-SM queue CTAs delay the
# router's persistent 148-CTA kernels by as much as they overlap; cfg4 4.71 vs 4.69 ms)
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q -x -k "complete or tick or queue or engine_clock or schedule or shard or bench or trace" 2>&1 | tail -2
for r in 1 2; do
  timeout 300 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/ov_cfg4.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ov_cfg4.json').read().strip().splitlines()[-1]);print('cfg4', round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['value']), {k:round(v,3) for k,v in d['stages_ms_per_tick'].items()})"
done
