cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -x -k "schedule or tick or select or dist or complete or shard" 2>&1 | tail -1
for lib in libchimera_sm100a.so libchimera_k6v1.so; do
  echo -n "$lib "; CHM_LIB=paper_2603_22206_b200/$lib timeout 300 python tools/select_bench.py --reps 20
done
