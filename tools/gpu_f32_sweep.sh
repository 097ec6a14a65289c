mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -5
for v in 34 24 33 44 26; do
  SF_SYM_F32_VARIANT=$v timeout 300 python tools/pair_perf.py --config c5 --reps 3 --mode 1 2>&1 | tail -1 | sed "s/^/f32v$v /"
done
timeout 300 python tools/pair_perf.py --config c5 --reps 3 --mode 0 2>&1 | tail -1 | sed "s/^/fp64 /"
