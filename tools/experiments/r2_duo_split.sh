#!/usr/bin/env bash
# duo fused QKV+attention: split issuers (warp 1 projection, warp 18 S / O;
# default) vs the single polling issuer (libchimera_ns.so: -DCHM_QA_DUO_SPLIT=0)
# (measured from a working tree and not kept: split issuers slower, 1.873 vs
# 1.728 ms at H = 768 and 0.390 vs 0.356 ms at H = 256; CHM_QA_DUO_SPLIT is not in
# the committed kernel)
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_gpu_router.py tests/test_gpu_attention.py tests/test_gpu_tick.py -q -x 2>&1 | tail -1
for r in 1 2; do
  for v in sm100a ns; do
    for h in 768 256; do
      echo -n "$v H=$h: "; CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 120 python tools/attn_micro.py --hidden $h --only fused --reps 10 2>&1 | tail -1
    done
  done
done
for c in cfg1 cfg4 cfg3; do for v in sm100a ns; do
  CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/ds_${c}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ds_${c}_$v.json').read().strip().splitlines()[-1]);st=d['stages_ms_per_tick'];print('$c $v', round(d['ms_per_step'],3), round(d['value']), 'qkv', round(st.get('qkv_attention',0),3), d['clocks']['sm_mhz'])"
done; done
