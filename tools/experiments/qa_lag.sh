# cta_group::1 fused QKV+attention: projection issue lag (S/O slotting latency)
export PYTHONUNBUFFERED=1
for l in 0 1 2 3 4 6; do echo "lag=$l"; CHM_QA_LAG=$l timeout 120 python tools/attn_micro.py --only fused --reps 20; done
for l in 0 3; do echo "lag=$l (repeat)"; CHM_QA_LAG=$l timeout 120 python tools/attn_micro.py --only fused --reps 20; done
