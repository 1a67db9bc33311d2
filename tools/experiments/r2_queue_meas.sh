#!/usr/bin/env bash
# K7 grid-wide path after the incremental commit: parity, stress (restored =
# full radix path; --chain = incremental path), ncu DRAM bytes of one chained call.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_gpu_queue_incremental.py tests/test_gpu_queue.py -q -x 2>&1 | tail -2
timeout 600 python tools/queue_stress.py --n 1048576 16777216 --steps 5
timeout 600 python tools/queue_stress.py --n 1048576 16777216 --steps 5 --chain
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q/chain16m.csv python tools/queue_stress.py --n 16777216 --steps 3 --chain > gpurun_out/q/ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q/full16m.csv python tools/queue_stress.py --n 16777216 --steps 1 > gpurun_out/q/ncu2.log 2>&1
tail -2 gpurun_out/q/ncu.log
