#!/usr/bin/env bash
# compute-sanitizer over the round-2 kernels: duo fused QKV+attention, flash v5,
# grid-wide queue (incremental path, staged merge, IF-node sections)
cd "$(dirname "$0")/../.."
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "test_qkv_attention or test_attention_matches or test_encoder_fused or long_prompts" > gpurun_out/san/${tool}_router.log 2>&1
  echo "$tool router rc=$? $(grep -c 'Hazard\|Invalid\|Error\b' gpurun_out/san/${tool}_router.log) $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY\|passed' gpurun_out/san/${tool}_router.log | tr '\n' ' ')"
done
timeout 900 $CS --tool memcheck --target-processes all --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "incremental or graph_replay" > gpurun_out/san/memcheck_queue.log 2>&1
echo "memcheck queue rc=$? $(grep 'ERROR SUMMARY\|passed' gpurun_out/san/memcheck_queue.log | tr '\n' ' ')"
