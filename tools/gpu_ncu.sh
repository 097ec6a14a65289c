set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 \
    -o gpurun_out/prof_pair_c5 python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/ncu.log
