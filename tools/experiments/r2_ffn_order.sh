#!/usr/bin/env bash
# fused FFN issue order: G1(c+2) before G2(c) (default) vs G2(c) first (CHM_FFN_TL bit 4)
# (measured from a working tree and not kept: no change, 0.572 vs 0.570 ms; the
# CHM_FFN_TL bit 4 order switch is not in the committed kernel)
cd "$(dirname "$0")/../.."
CHM_FFN_TL=4 timeout 300 python -m pytest tests/test_gpu_router.py -q -x -k "ffn_fused or encoder_matches or long_prompts" 2>&1 | tail -1
for r in 1 2; do
  for v in 0 4; do
    echo -n "order bits $v: "; CHM_FFN_TL=$v timeout 120 python tools/ffn_micro.py 2>&1 | grep fused
  done
done
CHM_FFN_TL=5 timeout 120 python tools/ffn_micro.py 2>&1 | sed -n 1,12p
for v in 0 4; do
  CHM_FFN_TL=$v timeout 300 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/fo_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/fo_$v.json').read().strip().splitlines()[-1]);print('cfg4 bits $v', round(d['ms_per_step'],3), round(d['value']), round(d['stages_ms_per_tick']['gemm'],3))"
done
