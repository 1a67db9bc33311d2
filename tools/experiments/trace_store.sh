# trace store: parity suite, micro-benchmark, ncu capture of the derive kernel
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_trace.py -x -q > gpurun_out/trace_pytest.txt 2>&1; tail -2 gpurun_out/trace_pytest.txt
timeout 300 python tools/trace_bench.py > gpurun_out/trace_bench.json 2> gpurun_out/trace_bench.err; cat gpurun_out/trace_bench.json
timeout 300 ncu --set full --clock-control none -k regex:derive_kernel -s 2 -c 1 -o gpurun_out/trace_derive python tools/trace_bench.py --reps 1 > gpurun_out/trace_ncu.log 2>&1
