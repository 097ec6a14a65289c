#!/bin/bash
# conflict-free j-pair staging in the packed FP32c kernel: probe of FFMA2 operand forms, FP32c tests, C3/C5 rates
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_probe2 tools/ffma2_probe2.cu && /tmp/ffma2_probe2 | tee gpurun_out/ffma2_probe2.txt
timeout 900 python -m pytest tests/test_gpu_fp32c_krylov.py tests/test_gpu_sym_waves.py tests/test_gpu_sym_split.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3
for c in c3 c5; do timeout 600 python tools/f32_variant.py $c | tee -a gpurun_out/f32_lay.jsonl; done
