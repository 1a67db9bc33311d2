# Shared-memory views keep the shared address space (STS/LDS instead of
# generic ST.E/LD.E): parity, fused kernel timeline + micro, GEMM micro, tick bench
export PYTHONUNBUFFERED=1
o=gpurun_out/ss
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest.txt 2>&1; tail -2 $o/pytest.txt
CHM_QA_DEBUG=11 timeout 60 python tools/attn_micro.py --timeline > $o/timeline.txt 2>&1
timeout 300 python tools/attn_micro.py > $o/attn_micro.txt 2>&1
timeout 300 python tools/gemm_micro.py > $o/gemm_micro.txt 2>&1
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
timeout 120 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/fused_ncu.csv 2>&1
echo "fused tensor% $(grep pct_of_peak $o/fused_ncu.csv | tail -1 | awk -F, '{print $NF}')"
for rep in 1 2; do timeout 400 python bench.py --no-cpu-baseline --no-e2e > $o/bench_cfg3_$rep.json 2> /dev/null; done
timeout 400 python bench.py --no-cpu-baseline --config cfg5 > $o/bench_cfg5.json 2>/dev/null
cat $o/attn_micro.txt $o/timeline.txt
for f in $o/bench_*.json; do echo "$f $(cut -c1-200 $f)"; done
