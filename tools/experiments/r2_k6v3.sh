#!/usr/bin/env bash
# K6 warp chain v3 (gate-free rows skip the reduction; runner-up tracking) vs v1
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/k6v3
timeout 900 python -m pytest tests -m gpu -q -x -k "schedule or tick or select or dist or complete or shard" > gpurun_out/k6v3/pytest.txt 2>&1; tail -2 gpurun_out/k6v3/pytest.txt
for r in 1 2; do
for lib in libchimera_sm100a.so libchimera_k6v1.so; do
  echo -n "$lib "; CHM_LIB=paper_2603_22206_b200/$lib timeout 300 python tools/select_bench.py --reps 20
done; done
for lib in libchimera_sm100a.so libchimera_k6v1.so; do
CHM_LIB=paper_2603_22206_b200/$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/k6v3/bench_cfg3_$lib.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/k6v3/bench_cfg3_$lib.json'));print('$lib', d['ms_per_step'], d['stages_ms_per_tick']['select'], d['clocks']['sm_mhz'])"
done
