#!/bin/bash
# packed FP32c kernel: per-i-point vs phase-grouped step, C5 and C3
mkdir -p gpurun_out
rm -f gpurun_out/f32p2_variants.log
for c in c5 c3; do
for v in ${VARIANTS:-134 234 224 233}; do
  SF_SYM_F32_VARIANT=$v timeout 600 python tools/f32_variant.py $c >> gpurun_out/f32p2_variants.log 2>&1
done; done
cat gpurun_out/f32p2_variants.log
SF_SYM_F32_VARIANT=${NCUV:-234} timeout 900 ncu --clock-control none -k regex:sym_task_kernel_f32 -s 2 -c 1 \
  --metrics gpu__time_duration.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,sm__warps_active.avg.per_cycle_active,launch__registers_per_thread \
  --csv python tools/f32_variant.py c5 > gpurun_out/f32p2_ncu.csv 2>&1; echo "ncu rc=$?"
grep -E "sym_task" gpurun_out/f32p2_ncu.csv | awk -F'","' '{print $13, $15}' 
