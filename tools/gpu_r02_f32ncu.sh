#!/bin/bash
# FP32 pipe probe (FFMA2 operand forms) + ncu --set full of the packed FP32c symmetric kernel at C3
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_probe2 tools/ffma2_probe2.cu && /tmp/ffma2_probe2 | tee gpurun_out/ffma2_probe2.txt
timeout 600 python tools/f32_variant.py c3 | tee gpurun_out/f32_c3_plain.json
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sym_task_kernel_f32p -c 1 \
    -f -o gpurun_out/prof_f32p_c3 python tools/f32_variant.py c3 > gpurun_out/ncu_f32p.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_f32p.log
ncu -i gpurun_out/prof_f32p_c3.ncu-rep --page raw --csv > gpurun_out/prof_f32p_c3_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_f32p_c3.ncu-rep --page source --csv > gpurun_out/prof_f32p_c3_source.csv 2>/dev/null
ls -la gpurun_out/prof_f32p_c3*
