# Warp-uniform MMA issue (elect.sync) in the fused QKV+attention, flash and
# GEMM issuers: parity, projection-only / full per-cycle tensor %, micro
# timings, tick bench.
export PYTHONUNBUFFERED=1
o=gpurun_out/iu
mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_router.py -x -q > $o/pytest.txt 2>&1; tail -3 $o/pytest.txt
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
CHM_QA_DEBUG=1 timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/proj.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/full.csv 2>&1
timeout 300 python tools/attn_micro.py > $o/attn_micro.txt 2>&1
timeout 300 python tools/gemm_micro.py > $o/gemm_micro.txt 2>&1
timeout 400 python bench.py --no-cpu-baseline > $o/bench_cfg3.json 2> $o/bench_cfg3.err
timeout 400 python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg3.csv python tools/profile_tick.py --ticks 3 > $o/launches.log 2>&1
ls $o
