#!/usr/bin/env bash
# fused H = 256 FFN: parity, then cfg1 / cfg4 ticks fused vs unfused (same box)
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_gpu_router.py -q -x -k "ffn_fused" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_attention.py tests/test_gpu_tick.py -q -x 2>&1 | tail -2
for c in cfg4 cfg1; do for f in 1 0; do
  CHM_FFN_FUSED=$f timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ffn_$c_$f.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ffn_$c_$f.json'));print('$c fused=$f', round(d['ms_per_step'],3), round(d['stages_ms_per_tick']['gemm'],3), d['clocks']['sm_mhz'])"
done; done
