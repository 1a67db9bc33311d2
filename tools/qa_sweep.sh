for c in 11 12 21 22 24; do for lag in 0 2 3; do
  echo "cluster=$c lag=$lag $(CHM_QA_CLUSTER=$c CHM_QA_LAG=$lag timeout -s KILL 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"
done; done
for c in 11 22; do echo "gemm-only cluster=$c $(CHM_QA_DEBUG=1 CHM_QA_CLUSTER=$c timeout -s KILL 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"; done
