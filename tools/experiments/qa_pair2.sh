# Pair-projection fused kernel (CHM_QA_PAIR=2: cta_group::2 projection + cta_group::1
# attention, 6 x 28 KB stages) vs the cta_group::1 kernel: parity, micro, ncu, tick A/B
export PYTHONUNBUFFERED=1
o=gpurun_out/qp2
mkdir -p $o
CHM_QA_PAIR=2 timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_router.py tests/test_gpu_tick.py -x -q > $o/pytest.txt 2>&1; tail -1 $o/pytest.txt
for p in 0 2 0 2; do echo "pair=$p $(CHM_QA_PAIR=$p timeout 60 python tools/attn_micro.py --only fused | tail -1)"; done > $o/micro.txt
echo "pair=2 proj-only $(CHM_QA_PAIR=2 CHM_QA_DEBUG=1 timeout 60 python tools/attn_micro.py --only fused | tail -1)" >> $o/micro.txt
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
CHM_QA_PAIR=2 timeout 120 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/ncu.csv 2>&1
echo "pair=2 tensor% $(grep pct_of_peak $o/ncu.csv | tail -1 | awk -F, '{print $NF}')" >> $o/micro.txt
CHM_QA_PAIR=2 CHM_QA_DEBUG=11 timeout 60 python tools/attn_micro.py --timeline | sed -n 3,5p >> $o/micro.txt
for rep in 1 2; do for p in 0 2; do
  echo "pair=$p $(CHM_QA_PAIR=$p timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["stages_ms_per_tick"]; print(round(d["ms_per_step"],2), round(d["value"]), d["clocks"]["sm_mhz"], round(s["qkv_attention"],2))')"
done; done > $o/bench.txt
cat $o/micro.txt $o/bench.txt
