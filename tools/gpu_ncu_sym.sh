timeout 300 python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/plain_sym.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sym_task -c 1 \
    -o gpurun_out/prof_sym_c5 python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/ncu_sym.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_sym.log
