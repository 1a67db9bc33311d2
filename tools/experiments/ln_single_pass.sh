# cluster-LN epilogue with one TMEM pass: parity, per-cycle, tick A/B vs the session-start build
export PYTHONUNBUFFERED=1
timeout 300 python -m pytest tests/test_gpu_router.py tests/test_gpu_tick.py -x -q 2>&1 | tail -1
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout 300 ncu --metrics $M --clock-control none --csv python tools/gemm_micro.py --reps 1 --only out_ln,ffn2_ln > gpurun_out/lnsp_ncu.csv 2>&1
for i in 1 2; do
  (cd _ab_old && timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['stages_ms_per_tick']['gemm'],2), round(d['stages_ms_per_tick']['qkv_attention'],2))")
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], round(d['stages_ms_per_tick']['gemm'],2), round(d['stages_ms_per_tick']['qkv_attention'],2))"
done
