#!/usr/bin/env bash
# duo vs PAIR fused kernel, same box: micro-benchmark and the cfg3 tick, twice
cd "$(dirname "$0")/../.."
for r in 1 2; do for d in 1 0; do
  echo -n "micro duo=$d: "; CHM_QA_DUO=$d timeout 60 python tools/attn_micro.py --hidden 768 --only fused --reps 50
done; done
for r in 1 2; do for d in 1 0; do
  CHM_QA_DUO=$d timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_duo$d.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_duo$d.json'));print('tick duo=$d', round(d['ms_per_step'],2), round(d['stages_ms_per_tick']['qkv_attention'],2), d['clocks']['sm_mhz'], d['clocks'].get('power_w'))"
done; done
