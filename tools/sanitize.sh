#!/usr/bin/env bash
# compute-sanitizer over the GPU parity tests (run on the GPU box):
#   memcheck  -- out-of-bounds / misaligned / leak checks on every kernel the
#                selected tests launch (router, K5-K7, monitor, trace, comm)
#   racecheck -- shared-memory hazards (selection, queue, monitor, trace)
#   synccheck -- barrier misuse (same set)
# Summaries go to gpurun_out/sanitize_*.log; tools/summarize_sanitize.py
# condenses them for profiles/.
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_SMALL="test_gpu_schedule or test_gpu_queue or test_gpu_complete or test_gpu_trace or test_gpu_predictor or test_gpu_engine_clock or test_gpu_evaluate"
SEL_ROUTER="test_gemm or test_attention or test_qkv_attention or test_encoder_routed_rows_only"
run() {  # tool, selection, log
  timeout 1500 $CS --tool "$1" --target-processes all --error-exitcode 97 \
    --print-limit 50 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$2" \
    > "$OUT/$3" 2>&1
  echo "$1 [$2] rc=$?" >> "$OUT/sanitize_summary.txt"
}
: > "$OUT/sanitize_summary.txt"
run memcheck "($SEL_SMALL) and not select_kat" sanitize_memcheck_small.log
run memcheck "$SEL_ROUTER" sanitize_memcheck_router.log
run racecheck "(test_gpu_schedule or test_gpu_queue or test_gpu_complete) and not select_kat" sanitize_racecheck.log
run synccheck "(test_gpu_schedule or test_gpu_queue or test_gpu_complete or test_gpu_trace) and not select_kat" sanitize_synccheck.log
cat "$OUT/sanitize_summary.txt"
