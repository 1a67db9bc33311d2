# derive-kernel chunk size sweep (entries per chunk), then the parity suite at the default
export PYTHONUNBUFFERED=1
for c in 256 512 1024 2048 4096; do echo "chunk $c"; CHM_TRACE_CHUNK=$c timeout 300 python tools/trace_bench.py --reps 20 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['derive_ms'], d['derive_GBps'], d['frac'])"; done > gpurun_out/trace_chunk.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_trace.py -x -q 2>&1 | tail -1 >> gpurun_out/trace_chunk.txt
