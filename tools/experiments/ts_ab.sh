# Q / P in TMEM (CHM_QA_TS=1) as the default? parity suite with it on, then a
# same-box interleaved tick A/B (3 reps each)
export PYTHONUNBUFFERED=1
o=gpurun_out/tsab
mkdir -p $o
CHM_QA_TS=1 timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_ts.txt 2>&1; tail -1 $o/pytest_ts.txt
for rep in 1 2 3; do
  for ts in 0 1; do
    echo "ts=$ts $(CHM_QA_TS=$ts timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],2), round(d["value"]), d["clocks"]["sm_mhz"], round(d["stages_ms_per_tick"]["qkv_attention"],2))')"
  done
done > $o/ab.txt
cat $o/ab.txt
