#!/usr/bin/env bash
# cluster-LN vs deferred LayerNorm with the duo fused kernel (cfg3, same box, twice)
cd "$(dirname "$0")/../.."
for r in 1 2; do for ln in cluster deferred; do
  timeout 300 python bench.py --layernorm $ln --no-cpu-baseline --no-e2e > gpurun_out/ln_$ln.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ln_$ln.json'));print('$ln', d['ms_per_step'], d['stages_ms_per_tick'].get('qkv_attention'), d['stages_ms_per_tick'].get('gemm'), d['clocks']['sm_mhz'])"
done; done
timeout 300 python -m pytest tests -m gpu -q -k "deferred or fold or layernorm" 2>&1 | tail -1
