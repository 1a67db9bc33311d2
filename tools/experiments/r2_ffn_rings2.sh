#!/usr/bin/env bash
# fused FFN (two issuers): W2 ring 3 slots (sm100a) vs 2 (a) vs W1 ring 6 slots (b)
# (measured from a working tree: every variant with the bias in global memory
# ran 0.52 ms vs 0.497 ms for the committed kernel -- the rings are not the
# bound once the two issuers are split; not kept)
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_gpu_router.py -q -x -k "ffn_fused or encoder_matches" 2>&1 | tail -1
for r in 1 2; do
  for v in sm100a a b; do
    echo -n "$v: "; CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 120 python tools/ffn_micro.py 2>&1 | grep fused
  done
done
for c in cfg4; do for v in sm100a a b; do
  CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/f3_${c}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/f3_${c}_$v.json').read().strip().splitlines()[-1]);print('$c $v', round(d['ms_per_step'],3), round(d['value']), round(d['stages_ms_per_tick']['gemm'],3))"
done; done
