#!/usr/bin/env bash
# K7 incremental path: shared-memory staged final merge; parity + 16.8M stress
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_queue_incremental.py tests/test_gpu_queue.py tests/test_gpu_tick.py tests/test_gpu_shard_queue.py tests/test_gpu_engine_clock.py -q -x 2>&1 | tail -1
for g in "" "--graph"; do timeout 600 python tools/queue_stress.py --n 16777216 --steps 5 --chain $g; done
mkdir -p gpurun_out/q; timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"final2_merge|fast_rounds|halo|heads_select" --csv --log-file gpurun_out/q/merge.csv python tools/queue_stress.py --n 16777216 --steps 2 --chain > /dev/null 2>&1
python tools/ncu_table.py gpurun_out/q/merge.csv | tail -4
CHM_QUEUE_COND=0 timeout 600 python tools/queue_stress.py --n 16777216 --steps 5 --chain --graph
CHM_QUEUE_COND=1 timeout 600 python tools/queue_stress.py --n 16777216 --steps 5 --chain --graph
