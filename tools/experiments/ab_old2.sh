# after the fold specialisation: same-box A/B vs the session-start build, plus GEMM parity
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_router.py -x -q 2>&1 | tail -1
for i in 1 2; do
  for c in cfg1 cfg3; do
    (cd _ab_old && timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old $c', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['stages_ms_per_tick'].items() if v > 0.05})")
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new $c', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['stages_ms_per_tick'].items() if v > 0.05})"
  done
done
