#!/usr/bin/env bash
# K7 grid-wide path: incremental fast path parity and the 16M-entry stress,
# restored (radix path) vs chained ticks (incremental path).
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_queue_incremental.py tests/test_gpu_queue.py -q -x 2>&1 | tail -15
timeout 600 python tools/queue_stress.py --n 1048576 16777216 --steps 5
timeout 600 python tools/queue_stress.py --n 1048576 16777216 --steps 5 --chain
