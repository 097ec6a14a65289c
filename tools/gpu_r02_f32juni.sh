#!/bin/bash
# packed FP32c kernel with the j slab's common c as a broadcast operand: tests + C3/C5 rates
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fp32c_krylov.py tests/test_gpu_sym_waves.py tests/test_gpu_sym_split.py tests/test_gpu_fullsize.py tests/test_gpu_mixed_orders.py -m gpu -q -x 2>&1 | tail -3
for c in c3 c5 c5; do timeout 600 python tools/f32_variant.py $c | tee -a gpurun_out/f32_juni.jsonl; done
for i in 1 2; do timeout 300 python tools/sym_aster_perf.py 1024; done
timeout 600 python tools/pair_perf.py --config c5 --reps 2
