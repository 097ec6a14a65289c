#!/bin/bash
# packed FP32c kernel after the conflict-free staging: launch-shape and unit sweep at C5
mkdir -p gpurun_out
for v in 344 334 343 444 234; do SF_SYM_F32_VARIANT=$v timeout 600 python tools/f32_variant.py c5 | tee -a gpurun_out/f32_sweep2.jsonl; done
for u in 1152 1280 1408; do SF_SYM_UNIT=$u timeout 600 python tools/f32_variant.py c5 | tee -a gpurun_out/f32_sweep2.jsonl; done
