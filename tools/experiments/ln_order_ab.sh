# deferred LayerNorm with the contiguous item order (the FOLD fused kernel then
# reuses each sequence's row affine across its heads) vs cluster LN
export PYTHONUNBUFFERED=1
o=gpurun_out/lnord
mkdir -p $o
for rep in 1 2; do
  for v in cluster deferred deferred_o1; do
    case $v in
      cluster) A="";; deferred) A="--layernorm deferred";; deferred_o1) A="--layernorm deferred"; export CHM_QA_ORDER=1;;
    esac
    echo "$v $(timeout 400 python bench.py --no-cpu-baseline --no-e2e $A 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d["stages_ms_per_tick"]; print(round(d["ms_per_step"],2), round(d["value"]), d["clocks"]["sm_mhz"], round(s["gemm"],2), round(s["qkv_attention"],2))')"
    unset CHM_QA_ORDER
  done
done > $o/ab.txt
for d in 0; do echo "fold micro order0 $(CHM_QA_ORDER=0 timeout 60 python tools/attn_micro.py --only fused | tail -1)"; done >> $o/ab.txt
cat $o/ab.txt
