# try_wait (default) vs test_wait spin for every mbarrier wait (-DCHM_SPIN_WAIT build
# in _ab_old/libspin.so): fused kernel timeline + micro, GEMM micro, tick bench
export PYTHONUNBUFFERED=1
o=gpurun_out/spin
mkdir -p $o
for lib in base spin; do
  L=paper_2603_22206_b200/libchimera_sm100a.so; [ $lib = spin ] && L=_ab_old/libspin.so
  echo "== $lib"
  CHM_LIB=$L timeout 120 python tools/attn_micro.py --only fused
  CHM_LIB=$L CHM_QA_DEBUG=11 timeout 60 python tools/attn_micro.py --timeline | sed -n 3,5p
  CHM_LIB=$L timeout 300 python tools/gemm_micro.py --only ffn 2>&1 | head -4
done > $o/micro.txt 2>&1
for lib in base spin base spin; do
  L=paper_2603_22206_b200/libchimera_sm100a.so; [ $lib = spin ] && L=_ab_old/libspin.so
  echo "$lib $(CHM_LIB=$L timeout 400 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | cut -c150-250)"
done > $o/bench_ab.txt
cat $o/micro.txt $o/bench_ab.txt
