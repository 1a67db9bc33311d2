# A/B against the session-start build (git worktree _ab_old @ fcf611e), same box, alternating
export PYTHONUNBUFFERED=1
for i in 1 2; do
  for c in cfg1 cfg3; do
    (cd _ab_old && timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old $c', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['stages_ms_per_tick'].items() if v > 0.05})")
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new $c', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k: round(v,3) for k,v in d['stages_ms_per_tick'].items() if v > 0.05})"
  done
done
