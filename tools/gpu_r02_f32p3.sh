#!/bin/bash
# packed FP32c kernel: owner sums in shared memory (128 registers -> 4 CTAs/SM) x unit size, C5
mkdir -p gpurun_out
rm -f gpurun_out/f32p3_variants.log
run() { echo "v=$1 unit=$2" >> gpurun_out/f32p3_variants.log
  SF_SYM_F32_VARIANT=$1 SF_SYM_UNIT=$2 timeout 600 python tools/f32_variant.py ${3:-c5} >> gpurun_out/f32p3_variants.log 2>&1; }
run 234 2048; run 334 2048; run 344 1024; run 344 1408; run 343 1024; run 444 1024; run 234 1024; run 344 1536
cat gpurun_out/f32p3_variants.log
