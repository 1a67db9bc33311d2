# L2 prefetch of the next tile's residual boxes in the residual / LN epilogues:
# GEMM micro (out_ln, ffn2_ln, out_resln, ffn2_resln) with per-cycle tensor %, A/B via CHM_LIB
export PYTHONUNBUFFERED=1
o=gpurun_out/rpl2
mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_router.py -x -q > $o/pytest.txt 2>&1; tail -1 $o/pytest.txt
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for lib in new old; do
  L=paper_2603_22206_b200/libchimera_sm100a.so; [ $lib = old ] && L=_ab_old/old_lib.so
  CHM_LIB=$L timeout 300 python tools/gemm_micro.py --only ln > $o/micro_$lib.txt 2>&1
  CHM_LIB=$L timeout 300 ncu --metrics $M --clock-control none --csv python tools/gemm_micro.py --reps 1 --only ln > $o/ncu_$lib.csv 2>&1
done
for lib in new old new old; do
  L=paper_2603_22206_b200/libchimera_sm100a.so; [ $lib = old ] && L=_ab_old/old_lib.so
  echo "$lib $(CHM_LIB=$L timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | cut -c150-260)"
done > $o/bench_ab.txt
cat $o/micro_*.txt $o/bench_ab.txt
