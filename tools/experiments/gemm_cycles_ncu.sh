export PYTHONUNBUFFERED=1
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum,lts__t_sectors_srcunit_tex.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg"
for d in 0 1 2; do
CHM_GEMM_DEBUG=$d timeout 300 ncu --metrics $M --clock-control none --csv python tools/gemm_micro.py --reps 1 --only ffn1_gelu,qkv,ffn2_resln,out_resln > gpurun_out/exp4_ncu_d$d.csv 2>&1
done
timeout 300 ncu --metrics $M --clock-control none --csv python tools/gemm_micro.py --reps 1 --only cublas > gpurun_out/exp4_ncu_cublas.csv 2>&1
timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/exp4_ncu_qa.csv 2>&1
CHM_QA_CLUSTER=11 timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/exp4_ncu_qa11.csv 2>&1
CHM_QA_DEBUG=1 timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > gpurun_out/exp4_ncu_qad1.csv 2>&1
python tools/gemm_micro.py --reps 100 > gpurun_out/exp4_energy.txt 2>&1
CHM_GEMM_DEBUG=2 python tools/gemm_micro.py --reps 100 --only ffn1_gelu,qkv >> gpurun_out/exp4_energy.txt 2>&1
