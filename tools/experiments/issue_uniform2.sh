# Warp-uniform producers too (fused, pair, GEMM); dbg 7 = the issue loop with no producer.
export PYTHONUNBUFFERED=1
o=gpurun_out/iu2
mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_gpu_router.py -x -q > $o/pytest.txt 2>&1; tail -2 $o/pytest.txt
CHM_QA_PAIR=1 timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > $o/pytest_pair.txt 2>&1; tail -2 $o/pytest_pair.txt
for d in 0 1 4 7; do echo "cg1 dbg=$d $(CHM_QA_DEBUG=$d timeout -s KILL 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"; done > $o/sweep.txt
for d in 0 1; do echo "pair dbg=$d $(CHM_QA_PAIR=1 CHM_QA_DEBUG=$d timeout -s KILL 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"; done >> $o/sweep.txt
cat $o/sweep.txt
timeout 300 python tools/gemm_micro.py > $o/gemm_micro.txt 2>&1
timeout 400 python bench.py --no-cpu-baseline > $o/bench_cfg3.json 2> $o/bench_cfg3.err
