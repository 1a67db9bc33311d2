# cfg3: session-start build vs deferred LN vs cluster LN (same box, alternating)
export PYTHONUNBUFFERED=1
for i in 1 2; do
  (cd _ab_old && timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['stages_ms_per_tick']['gemm'],2), round(d['stages_ms_per_tick']['qkv_attention'],2))")
  for ln in deferred cluster; do
    timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --layernorm $ln 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$ln', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['stages_ms_per_tick']['gemm'],2), round(d['stages_ms_per_tick']['qkv_attention'],2))"
  done
done
