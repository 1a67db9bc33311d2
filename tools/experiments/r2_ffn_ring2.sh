#!/usr/bin/env bash
# fused FFN: W2 ring of 3 slots (default) vs 2 (libchimera_w2.so: tools/build_variant.py
# libchimera_w2.so -DCHM_FFN_SLOTS2=2); parity; per-chunk timeline; ticks
# (measured from a working tree and not kept: 0.585 vs 0.586 ms with the single
# issuer; CHM_FFN_SLOTS2 is not in the committed kernel)
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_gpu_router.py -q -x -k "ffn_fused or encoder_matches or long_prompts" 2>&1 | tail -1
for r in 1 2; do
  for v in sm100a w2; do
    echo -n "$v: "; CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 120 python tools/ffn_micro.py 2>&1 | grep fused
  done
done
CHM_FFN_TL=1 timeout 120 python tools/ffn_micro.py 2>&1 | sed -n 1,10p
for c in cfg4 cfg1; do for v in sm100a w2; do
  CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/fr_${c}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/fr_${c}_$v.json').read().strip().splitlines()[-1]);print('$c $v', round(d['ms_per_step'],3), round(d['value']), round(d['stages_ms_per_tick']['gemm'],3))"
done; done
