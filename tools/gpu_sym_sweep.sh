timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -2
for cfg in "SF_SYM_MINB=4" "SF_SYM_MINB=3"; do
  env $cfg timeout 300 python tools/pair_perf.py --config c5 --reps 2 2>&1 | tail -1 | sed "s/^/$cfg /"
done
