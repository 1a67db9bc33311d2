# fused QKV+attention item order (interleaved vs contiguous), cfg1 (no fold) and cfg3 (fold), same box
export PYTHONUNBUFFERED=1
for i in 1 2; do for o in 0 1; do for c in cfg1 cfg3; do
  CHM_QA_ORDER=$o timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('order=$o $c', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['stages_ms_per_tick']['qkv_attention'],3), round(d['stages_ms_per_tick']['gemm'],3))"
done; done; done
