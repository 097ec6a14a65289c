#!/bin/bash
# j-pair packed FFMA2 FP32c kernel (sym_task_kernel_f32p) vs the scalar FP32c kernel, C5 and C3,
# then targeted ncu metrics of the packed kernel at C5 (one wave launch)
mkdir -p gpurun_out
for c in c5 c3; do
for v in 34 134 124 133; do
  SF_SYM_F32_VARIANT=$v timeout 600 python tools/f32_variant.py $c >> gpurun_out/f32p_variants.log 2>&1
done; done
cat gpurun_out/f32p_variants.log
SF_SYM_F32_VARIANT=${NCUV:-134} timeout 900 ncu --clock-control none -k regex:sym_task_kernel_f32 -s 2 -c 1 \
  --metrics gpu__time_duration.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,sm__warps_active.avg.per_cycle_active,launch__registers_per_thread \
  --csv python tools/f32_variant.py c5 > gpurun_out/f32p_ncu.csv 2>&1; echo "ncu rc=$?"
grep -E "sym_task|Metric" gpurun_out/f32p_ncu.csv | cut -c1-400 | tail -20
