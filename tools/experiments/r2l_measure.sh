#!/usr/bin/env bash
# Round-2 last pass after the two-issuer fused FFN: GPU suite, smoke, bench
# lines for every config + the reference arm, cfg1 / cfg4 launch lists
export PYTHONUNBUFFERED=1
o=gpurun_out/${OUT:-r2l}
mkdir -p $o
nvidia-smi -L > $o/smi.txt
CHM_PARITY_LOG=$o/parity.jsonl timeout 1500 python -m pytest tests -m gpu -q -rs > $o/pytest_gpu.txt 2>&1; tail -2 $o/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; tail -1 $o/smoke.txt
timeout 600 python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
for c in cfg1 cfg2 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.json 2> $o/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg4.csv python tools/profile_tick.py --config cfg4 --ticks 3 > $o/launches4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_cfg1.csv python tools/profile_tick.py --config cfg1 --ticks 3 > $o/launches1.log 2>&1
ls $o | wc -l
