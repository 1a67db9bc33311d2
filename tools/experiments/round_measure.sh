# Round-end measurement pass: parity suite, bench lines for every config, the
# reference arm, the cfg3 launch list and a --set full capture of one layer's
# router kernels (qkv_attention + out-proj / FFN1 / FFN2 GEMMs) inside the tick.
export PYTHONUNBUFFERED=1
o=gpurun_out/${OUT:-rm}
mkdir -p $o
nvidia-smi -L > $o/smi.txt
timeout 900 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; tail -2 $o/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; tail -1 $o/smoke.txt
timeout 400 python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
for c in cfg1 cfg2 cfg4 cfg5; do timeout 400 python bench.py --config $c --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err; done
for c in cfg1 cfg4; do timeout 400 python bench.py --config $c --graph --no-cpu-baseline --no-e2e > $o/bench_${c}_graph.json 2> $o/bench_${c}_graph.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.json 2> $o/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg3.csv python tools/profile_tick.py --ticks 3 > $o/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|qkv_attention" -s 52 -c 4 -o $o/full_cfg3 python tools/profile_tick.py --ticks 2 > $o/full.log 2>&1
timeout 300 python tools/trace_bench.py > $o/trace_bench.json 2> $o/trace_bench.err
ls $o
