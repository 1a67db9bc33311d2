# projection-only rates: cta_group::1 fused kernel vs the cta_group::2 pair kernel (CHM_QA_DEBUG=1)
export PYTHONUNBUFFERED=1
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
CHM_QA_DEBUG=1 timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/proj_cg1.csv 2>&1
CHM_QA_PAIR=1 CHM_QA_DEBUG=1 timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/proj_cg2.csv 2>&1
