# After the warp-uniform issue change: issue lag, cluster shape and TS sweeps of the fused kernel
export PYTHONUNBUFFERED=1
o=gpurun_out/ql2
mkdir -p $o
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for cfg in "21 0 0 0" "21 1 0 0" "21 2 0 0" "21 3 0 0" "21 0 2 0" "11 0 0 0" "12 0 0 0" "22 0 0 0" "22 2 0 0" "21 0 0 1" "21 2 0 1"; do
  set -- $cfg
  CHM_QA_CLUSTER=$1 CHM_QA_LAG=$2 CHM_QA_DEBUG=$3 CHM_QA_TS=$4 timeout 120 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/run.csv 2>&1
  echo "cluster=$1 lag=$2 dbg=$3 ts=$4 $(grep pct_of_peak $o/run.csv | tail -1 | awk -F, '{print $NF}') $(grep gpu__time_duration $o/run.csv | tail -1 | awk -F, '{print $NF}') | $(CHM_QA_CLUSTER=$1 CHM_QA_LAG=$2 CHM_QA_DEBUG=$3 CHM_QA_TS=$4 timeout 60 python tools/attn_micro.py --only fused 2>&1 | tail -1)"
done > $o/summary.txt
cat $o/summary.txt
