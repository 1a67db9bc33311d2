#!/usr/bin/env bash
# fused QKV+attention (PAIR) per-item timeline of CTA 0 + kernel time
cd "$(dirname "$0")/../.."
timeout 120 python tools/attn_micro.py --only fused --reps 20
CHM_QA_DEBUG=11 timeout 120 python tools/attn_micro.py --timeline
