export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_router.py -x -q > gpurun_out/exp5_pytest.txt 2>&1; tail -2 gpurun_out/exp5_pytest.txt
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,sm__cycles_elapsed.avg"
timeout 300 ncu --metrics $M --clock-control none --csv python tools/gemm_micro.py --reps 1 --only out_resln,ffn2_resln,out_ln > gpurun_out/exp5_ncu.csv 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp5_bench_fused.json 2> gpurun_out/exp5_bench.err
timeout 300 python bench.py --no-cpu-baseline --attention unfused > gpurun_out/exp5_bench_unfused.json 2>> gpurun_out/exp5_bench.err
