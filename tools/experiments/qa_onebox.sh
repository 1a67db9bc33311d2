# fused QKV+attention, one 3-part W box per CTA per stage: parity, projection-only and full rates, tick
export PYTHONUNBUFFERED=1
timeout 120 python -m pytest tests/test_gpu_attention.py -x -q 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_router.py -x -q 2>&1 | tail -1
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
CHM_QA_DEBUG=1 timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/onebox_proj.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/onebox_full.csv 2>&1
for i in 1 2; do timeout 120 python tools/attn_micro.py --only fused --reps 20; done
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tick', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks'].get('energy_j_per_step'), round(d['stages_ms_per_tick']['qkv_attention'],2))"; done
