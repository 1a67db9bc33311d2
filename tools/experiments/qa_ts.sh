# fused QKV+attention with Q / P from tensor memory (CHM_QA_TS=1): parity, micro, tick A/B
export PYTHONUNBUFFERED=1
CHM_QA_TS=1 timeout 120 python -m pytest tests/test_gpu_attention.py -x -q -k "qkv or fused" 2>&1 | tail -2
CHM_QA_TS=1 timeout 300 python -m pytest tests/test_gpu_router.py -x -q 2>&1 | tail -2
for t in 0 1 0 1; do echo "ts=$t"; CHM_QA_TS=$t timeout 120 python tools/attn_micro.py --only fused --reps 20; done
for t in 0 1 0 1; do CHM_QA_TS=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ts=$t', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks'].get('energy_j_per_step'), round(d['stages_ms_per_tick']['qkv_attention'],2))"; done
