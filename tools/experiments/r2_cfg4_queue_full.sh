#!/usr/bin/env bash
# cfg4 K7 queue kernel: --set full capture with source, plus cfg3 / cfg5 bench
# lines with the associative last layer's algorithmic FLOP accounting
export PYTHONUNBUFFERED=1
o=gpurun_out/${OUT:-r2j}
mkdir -p $o
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"queue_kernel" -s 2 -c 1 -o $o/full_queue_cfg4 python tools/profile_tick.py --config cfg4 --ticks 2 > $o/fullq.log 2>&1
tail -2 $o/fullq.log
for c in cfg3 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err; done
ls $o
