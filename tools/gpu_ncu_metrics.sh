# Targeted ncu counters for the dominant kernels: instruction mix,
# FP64 pipe activity and DRAM bytes.  Each command first runs without ncu.
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 300 python tools/pair_perf.py --config c5 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:sym_task -c 1 --csv \
    python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/ncu_metrics_sym_c5.csv 2>&1
echo "sym rc=$?"
timeout 300 python tools/matvec_profile.py c4 > /dev/null 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"cross_task|dl_task|sym_task|pair_kernel" --csv \
    python tools/matvec_profile.py c4 > gpurun_out/ncu_metrics_c4.csv 2>&1
echo "c4 rc=$?"
