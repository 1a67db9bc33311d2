export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_attention.py -x -q > gpurun_out/exp3_pytest.txt 2>&1
tail -5 gpurun_out/exp3_pytest.txt
python tools/gemm_micro.py --reps 20 > gpurun_out/exp3_micro.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/exp3_bench.json 2> gpurun_out/exp3_bench.err
cat gpurun_out/exp3_micro.txt gpurun_out/exp3_bench.json
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp3_pytest_all.txt 2>&1; tail -3 gpurun_out/exp3_pytest_all.txt
