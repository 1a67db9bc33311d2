#!/usr/bin/env bash
# r2m bench lines (final HEAD: cls_pool lookahead, flash v6 O+l merge)

export PYTHONUNBUFFERED=1
o=gpurun_out/r2m
mkdir -p $o
timeout 600 python bench.py > $o/bench_cfg3.json 2> $o/bench_cfg3.err
for c in cfg1 cfg2 cfg4 cfg5; do timeout 600 python bench.py --config $c --no-cpu-baseline > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_ref.json 2> $o/bench_ref.err
ls $o | wc -l
