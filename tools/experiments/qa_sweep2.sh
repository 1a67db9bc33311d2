# Cluster-shape sweep of the fused QKV+attention kernel after the warp-uniform
# issue change: full kernel, projection only (dbg 1), projection without loads (dbg 4)
export PYTHONUNBUFFERED=1
o=gpurun_out/qs2
mkdir -p $o
for c in 11 12 21 22 24; do
  for d in 0 1 4; do
    echo "cluster=$c dbg=$d $(CHM_QA_DEBUG=$d CHM_QA_CLUSTER=$c timeout -s KILL 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"
  done
done > $o/sweep.txt
for c in 21 22; do for lag in 2 3; do
  echo "cluster=$c lag=$lag $(CHM_QA_CLUSTER=$c CHM_QA_LAG=$lag timeout -s KILL 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"
done; done >> $o/sweep.txt
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_bytes.sum.per_second,l1tex__m_xbar2l1tex_read_bytes.sum.per_second"
for c in 21 22; do
CHM_QA_DEBUG=1 CHM_QA_CLUSTER=$c timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/proj_$c.csv 2>&1
CHM_QA_CLUSTER=$c timeout 300 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/full_$c.csv 2>&1
done
cat $o/sweep.txt
