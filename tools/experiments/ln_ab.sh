export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_tick.py -x -q > gpurun_out/exp6_pytest.txt 2>&1; tail -2 gpurun_out/exp6_pytest.txt
for i in 1 2; do for ln in deferred cluster; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 --layernorm $ln > gpurun_out/exp6_$ln$i.json 2>> gpurun_out/exp6.err
done; done
