# Projection-only rate of the fused kernel, dissected: dbg 1 (full pipeline),
# 4 (no loads), 7 (no producer), 8 (+ accumulators 256 apart), 9 (+ local
# commits), 10 (+ no accumulator handshake, epilogue idle). ncu per-cycle tensor %.
export PYTHONUNBUFFERED=1
o=gpurun_out/qd
mkdir -p $o
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
for d in 1 4 7 8 9 10; do
  CHM_QA_DEBUG=$d timeout 120 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/d$d.csv 2>&1
  echo "dbg=$d $(grep pct_of_peak $o/d$d.csv | tail -1 | awk -F, '{print $NF}') $(grep gpu__time_duration $o/d$d.csv | tail -1 | awk -F, '{print $NF}')"
done > $o/summary.txt
CHM_QA_CLUSTER=11 CHM_QA_DEBUG=10 timeout 120 ncu --metrics $M --clock-control none --csv python tools/attn_micro.py --reps 1 --only fused > $o/c11_d10.csv 2>&1
echo "c11 dbg=10 $(grep pct_of_peak $o/c11_d10.csv | tail -1 | awk -F, '{print $NF}')" >> $o/summary.txt
CHM_QA_DEBUG=7 timeout 300 ncu --set full --import-source on --clock-control none -k regex:qkv_attention -s 3 -c 1 -o $o/d7_full python tools/attn_micro.py --reps 1 --only fused > $o/d7_full.log 2>&1
cat $o/summary.txt
