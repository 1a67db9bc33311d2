#!/usr/bin/env bash
# embedding + LayerNorm kernel: tokens per warp 1 / 2 / 4 (CHM_EMBED_ROWS), cfg3 and cfg4
cd "$(dirname "$0")/../.."
for c in cfg3 cfg4; do for r in 1 2 4; do
  CHM_EMBED_ROWS=$r timeout 300 ncu --metrics gpu__time_duration.sum -k regex:embed_ln --clock-control none --csv --log-file gpurun_out/emb_$c_$r.csv python tools/profile_tick.py --config $c --ticks 1 > /dev/null 2>&1
  echo -n "$c rows $r: "; python tools/ncu_table.py gpurun_out/emb_$c_$r.csv | tail -1
done; done
CHM_EMBED_ROWS=4 timeout 300 python -m pytest tests/test_gpu_router.py -q -x -k "encoder" 2>&1 | tail -1
