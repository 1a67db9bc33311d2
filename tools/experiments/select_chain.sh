# K6 warp-speculative chain: parity suite + stage timings at cfg1/cfg3/cfg4
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/sel_pytest.txt 2>&1; tail -2 gpurun_out/sel_pytest.txt
for c in cfg3 cfg1 cfg4; do
timeout 300 python bench.py --no-cpu-baseline --config $c > gpurun_out/sel_bench_$c.json 2>> gpurun_out/sel_bench.err
done
