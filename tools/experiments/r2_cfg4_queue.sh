#!/usr/bin/env bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/c4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4/q_cfg4.csv python tools/profile_tick.py --config cfg4 --ticks 2 > gpurun_out/c4/q.log 2>&1
tail -1 gpurun_out/c4/q.log
