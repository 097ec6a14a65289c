timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/pair_perf.py --config c3 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_task -c 1 \
    -o gpurun_out/prof_sym_c3 python tools/pair_perf.py --config c3 --reps 1 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu.log
