timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -1
for v in 224 124 24 233 223 232; do
  SF_SYM_VARIANT=$v timeout 300 python tools/pair_perf.py --config c5 --reps 2 2>&1 | tail -1 | sed "s/^/v$v /"
done
