#!/usr/bin/env bash
# K6 warp chain v2 (runner-up tracking) vs v1 (full argmin per row): parity + ns/decision
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/k6v2
timeout 900 python -m pytest tests -m gpu -q -x -k "schedule or tick or select or dist or complete" > gpurun_out/k6v2/pytest.txt 2>&1; tail -2 gpurun_out/k6v2/pytest.txt
for r in 1 2; do
for lib in libchimera_sm100a.so libchimera_k6v1.so; do
  echo -n "$lib "; CHM_LIB=paper_2603_22206_b200/$lib timeout 300 python tools/select_bench.py --reps 20
done; done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/k6v2/bench_cfg3.json 2>&1
python -c "import json;d=json.load(open('gpurun_out/k6v2/bench_cfg3.json'));print(d['ms_per_step'], d['stages_ms_per_tick']['select'])"
