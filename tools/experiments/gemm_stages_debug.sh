export PYTHONUNBUFFERED=1
o=gpurun_out/exp2.txt
echo "== base" > $o; python tools/gemm_micro.py --reps 40 >> $o 2>&1
echo "== stages6" >> $o; CHM_GEMM_STAGES=6 python tools/gemm_micro.py --reps 40 --only qkv,ffn1 >> $o 2>&1
echo "== dbg1" >> $o; CHM_GEMM_DEBUG=1 python tools/gemm_micro.py --reps 40 --only qkv,ffn1,ln >> $o 2>&1
echo "== dbg2" >> $o; CHM_GEMM_DEBUG=2 python tools/gemm_micro.py --reps 40 --only qkv,ffn1,ln >> $o 2>&1
echo "== stages6 dbg2" >> $o; CHM_GEMM_STAGES=6 CHM_GEMM_DEBUG=2 python tools/gemm_micro.py --reps 40 --only qkv,ffn1 >> $o 2>&1
echo "== base again" >> $o; python tools/gemm_micro.py --reps 40 >> $o 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,launch__grid_size,launch__cluster_dim_x,launch__shared_mem_per_block_dynamic --clock-control none --csv python tools/gemm_micro.py --reps 1 > gpurun_out/exp2_ncu.csv 2>&1
