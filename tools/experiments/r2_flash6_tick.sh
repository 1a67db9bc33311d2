#!/usr/bin/env bash
# full GPU suite with flash v6 as the default, then the cfg5 tick with v6 and v5
export PYTHONUNBUFFERED=1
o=gpurun_out/${OUT:-r2g}
mkdir -p $o
timeout 1200 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; tail -2 $o/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; tail -1 $o/smoke.txt
for r in 1 2; do
  for v in 6 5; do
    CHM_FLASH=$v timeout 400 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > $o/bench_cfg5_v$v.json 2> $o/bench_cfg5_v$v.err
    python - "$o/bench_cfg5_v$v.json" $v <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
sec=[x for x in d["roofline"]["secondary"] if "flash" in x["kernel"]]
print("v"+sys.argv[2], round(d["value"]), "dec/s", round(d["ms_per_step"],2), "ms tick", "attn", round(d["stages_ms_per_tick"]["attention"],2), "ms", "clock", d["clocks"]["sm_mhz"])
PY
  done
done
