#!/usr/bin/env bash
# fused FFN with E1 in two k-block halves (each signalled; default) vs one whole-chunk E1
# (libchimera_one.so: the two-issuer commit, built with tools/build_variant.py from a stash)
# (measured from a working tree, not kept: 0.499 vs 0.499 ms; the per-chunk
# stamps show the G1 stream gated by the one-chunk W1 ring: G1(c+1) issues ~2.4k
# cycles after G1(c), 1,024 of MMA plus the W1 reload)
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_gpu_router.py tests/test_gpu_tick.py -q -x -k "ffn_fused or encoder_matches or long_prompts or routed or cfg1 or cfg4" 2>&1 | tail -1
for r in 1 2; do
  for v in sm100a one; do
    echo -n "$v: "; CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 120 python tools/ffn_micro.py 2>&1 | grep fused
  done
done
CHM_FFN_TL=1 timeout 120 python tools/ffn_micro.py 2>&1 | sed -n 1,10p
for c in cfg4 cfg1; do for v in sm100a one; do
  CHM_LIB=paper_2603_22206_b200/libchimera_$v.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/f2_${c}_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/f2_${c}_$v.json').read().strip().splitlines()[-1]);print('$c $v', round(d['ms_per_step'],3), round(d['value']), round(d['stages_ms_per_tick']['gemm'],3))"
done; done
