#!/usr/bin/env bash
# two-issuer fused FFN: W1 ring 6 slots (b1 table cut to F <= 1024) vs 4 (libchimera_r4.so)
# (measured from a working tree, not kept: 0.507 vs 0.500 ms, cfg4 4.49 vs 4.46 ms)
cd "$(dirname "$0")/../.."
for r in 1 2; do
  for v in sm100a r4; do
    echo -n "$v: "; CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 120 python tools/ffn_micro.py 2>&1 | grep fused
  done
done
for c in cfg4 cfg1; do for v in sm100a r4; do
  CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/f6_${c}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/f6_${c}_$v.json').read().strip().splitlines()[-1]);print('$c $v', round(d['ms_per_step'],3), round(d['value']))"
done; done
