#!/usr/bin/env bash
# associative last layer (cls_pool.cu): parity, then cfg3 / cfg5 ticks with it on / off
export PYTHONUNBUFFERED=1
o=gpurun_out/${OUT:-r2h}
mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_tick.py -m gpu -q -x -s 2>&1 | grep -E "cls_pool|passed|failed|Error|error" | tail -8
for r in 1 2; do
  for c in cfg3 cfg5; do
    for v in 1 0; do
      CHM_CLS_POOL=$v timeout 400 python bench.py --config $c --no-cpu-baseline --no-e2e > $o/bench_${c}_pool$v.json 2> $o/bench_${c}_pool$v.err
      python - "$o/bench_${c}_pool$v.json" "$c pool=$v" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
st=d["stages_ms_per_tick"]
print(sys.argv[2], round(d["value"]), "dec/s", round(d["ms_per_step"],2), "ms", "gemm", round(st["gemm"],2), "attn", round(st["attention"],2), "clock", d["clocks"]["sm_mhz"], "J", d["clocks"].get("energy_j_per_step"))
PY
    done
  done
done
