#!/usr/bin/env bash
# cls_pool: pass 1 of sequence i + 1 before pass 2 of i (default) vs strictly
# per sequence (libchimera_old.so, the previous commit)
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_tick.py -q -x -k "cls_pool or encoder or routed or full_tick" 2>&1 | tail -1
for c in cfg3 cfg4; do for v in sm100a old; do
  CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/cp_${c}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/cp_${c}_$v.json').read().strip().splitlines()[-1]);print('$c $v', round(d['ms_per_step'],3), round(d['value']), 'pool', round(d['stages_ms_per_tick']['attention'],4))"
done; done
