timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -1
for v in 24 32 33 34 26 28 44; do
  SF_SYM_F32_VARIANT=$v timeout 300 python tools/pair_perf.py --config c5 --reps 3 --mode 1 2>&1 | tail -1 | sed "s/^/f32v$v /"
done
