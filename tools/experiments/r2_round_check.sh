bash tools/experiments/r2_flash.sh > gpurun_out/flash.log 2>&1
CHM_PARITY_LOG=gpurun_out/parity4.jsonl timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -v "^{" | tail -8 > gpurun_out/t9.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --target-processes all --print-limit 20 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "(test_gpu_schedule or test_gpu_queue or test_gpu_complete) and not select_kat" > gpurun_out/sanitize_racecheck2.log 2>&1
bash tools/experiments/r2_bench_all.sh > gpurun_out/bench_all.log 2>&1
cat gpurun_out/flash.log gpurun_out/t9.log gpurun_out/bench_all.log; grep "ERROR SUMMARY\|passed" gpurun_out/sanitize_racecheck2.log
