# cta_group::2 fused QKV+attention kernel: parity (kernel-level + encoder), micro by issue lag
export PYTHONUNBUFFERED=1
CHM_QA_PAIR=1 timeout 120 python -m pytest tests/test_gpu_attention.py -x -q -k "qkv or fused" 2>&1 | tail -2
CHM_QA_PAIR=1 timeout 300 python -m pytest tests/test_gpu_router.py -x -q 2>&1 | tail -2
echo "cg1"; CHM_QA_PAIR=0 timeout 120 python tools/attn_micro.py --only fused
for l in 0 1 2 3; do echo "pair lag=$l"; CHM_QA_PAIR=1 CHM_QAP_LAG=$l timeout 120 python tools/attn_micro.py --only fused; done
echo "cg1"; CHM_QA_PAIR=0 timeout 120 python tools/attn_micro.py --only fused
