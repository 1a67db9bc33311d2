# Same-box A/B after the issue fix: cluster vs deferred LayerNorm, TS fused kernel
export PYTHONUNBUFFERED=1
o=gpurun_out/lnab2
mkdir -p $o
for rep in 1 2; do
  timeout 400 python bench.py --no-cpu-baseline --no-e2e > $o/cluster_$rep.json 2>/dev/null
  timeout 400 python bench.py --no-cpu-baseline --no-e2e --layernorm deferred > $o/deferred_$rep.json 2>/dev/null
  CHM_QA_TS=1 timeout 400 python bench.py --no-cpu-baseline --no-e2e > $o/ts_$rep.json 2>/dev/null
done
for f in $o/*.json; do echo "$f $(python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), round(d['value']), d['clocks']['sm_mhz'], d['clocks'].get('energy_j_per_step'), {k: round(v,2) for k,v in d['stages_ms_per_tick'].items() if v > 0.3})
")"; done
