# Provably warp-uniform role branches (sm100::warp_id): parity, projection
# dissection, micro timings, tick bench.
export PYTHONUNBUFFERED=1
o=gpurun_out/${OUT:-uw}
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.txt 2>&1; tail -2 $o/pytest.txt
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for d in 0 1 4 7 10; do
  CHM_QA_DEBUG=$d timeout 120 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/d$d.csv 2>&1
  echo "dbg=$d $(grep pct_of_peak $o/d$d.csv | tail -1 | awk -F, '{print $NF}') $(grep gpu__time_duration $o/d$d.csv | tail -1 | awk -F, '{print $NF}')"
done > $o/summary.txt
cat $o/summary.txt
timeout 300 python tools/attn_micro.py > $o/attn_micro.txt 2>&1
CHM_QA_PAIR=1 timeout 300 python tools/attn_micro.py --only fused > $o/attn_micro_pair.txt 2>&1
timeout 300 python tools/gemm_micro.py > $o/gemm_micro.txt 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv python tools/gemm_micro.py --reps 1 > $o/gemm_ncu.csv 2>&1
timeout 400 python bench.py --no-cpu-baseline > $o/bench_cfg3.json 2> $o/bench_cfg3.err
timeout 400 python bench.py --config cfg1 --no-cpu-baseline > $o/bench_cfg1.json 2> $o/bench_cfg1.err
