#!/usr/bin/env bash
# Round-2 bench lines for every BASELINE configuration + the reference arm.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/r2b
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2b/bench_$c.json 2> gpurun_out/r2b/bench_$c.err
  echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b/bench_ref.json 2> gpurun_out/r2b/bench_ref.err
echo "ref rc=$?"
