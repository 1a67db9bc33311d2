# energy per launch (NVML cumulative counter over ~2 s per case) and the bench's power / energy fields
export PYTHONUNBUFFERED=1
python tools/gemm_micro.py --seconds 2 --only cublas,qkv,out_ln,ffn1_gelu,ffn2_ln > gpurun_out/energy_gemm.txt 2>&1
cat gpurun_out/energy_gemm.txt
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/energy_bench.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/energy_bench.json')); print(d['value'], d['ms_per_step'], d['clocks'])"
