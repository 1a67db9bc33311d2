#!/usr/bin/env bash
# compute-sanitizer over the last round-2 kernels: flash v6 (ping-pong tiles,
# two issuers), the associative last layer (cls_pool, build_bd), the K7 radix
# pass with per-warp slices
cd "$(dirname "$0")/../.."
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san2
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "test_attention_matches or long_prompts or cls_pool or encoder_matches" > gpurun_out/san2/${tool}_router.log 2>&1
  echo "$tool router rc=$? $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY\|passed' gpurun_out/san2/${tool}_router.log | tr '\n' ' ')"
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "test_queue_matches_reference or test_queue_order_random_large and not 2000000" > gpurun_out/san2/${tool}_queue.log 2>&1
  echo "$tool queue rc=$? $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY\|passed' gpurun_out/san2/${tool}_queue.log | tr '\n' ' ')"
done
