# projection-only rate of the fused kernel: accumulators 192 vs 256 TMEM columns apart
export PYTHONUNBUFFERED=1
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for d in 4 5 6; do CHM_QA_DEBUG=$d timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/align_d$d.csv 2>&1; done
