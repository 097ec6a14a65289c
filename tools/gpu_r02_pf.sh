#!/bin/bash
# single-shot slab meta load + next-slab L1 prefetch: tests, FP64 C5/C2 and FP32c C3/C5 rates
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fp32c_krylov.py tests/test_gpu_sym_waves.py tests/test_gpu_sym_split.py tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -3
for i in 1 2; do timeout 300 python tools/sym_aster_perf.py 1024; done
timeout 600 python tools/pair_perf.py --config c5 --reps 2
timeout 600 python tools/pair_perf.py --config c3 --reps 3
for c in c3 c5; do timeout 600 python tools/f32_variant.py $c | tee -a gpurun_out/f32_pf.jsonl; done
