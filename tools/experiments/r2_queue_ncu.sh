#!/usr/bin/env bash
# K7 16.8M-entry chained tick: per-launch DRAM bytes / time (ncu, cold, serialised)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/q
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q/chain16m_r2.csv python tools/queue_stress.py --n 16777216 --steps 2 --chain > gpurun_out/q/ncu_r2.log 2>&1
tail -1 gpurun_out/q/ncu_r2.log
