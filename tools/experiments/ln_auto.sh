# LN path choice by hidden size: router parity, then cfg1 (H=256) and cfg3 (H=768) A/B
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_router.py -x -q 2>&1 | tail -1
for i in 1 2; do for ln in auto deferred; do
timeout 300 python bench.py --config cfg1 --no-cpu-baseline --no-e2e --steps 50 --layernorm $ln > gpurun_out/lnauto_cfg1_$ln$i.json 2>/dev/null
done; done
