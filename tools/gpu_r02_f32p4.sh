#!/bin/bash
# new FP32c default (packed kernel, 1408-point units): GPU suite + C5/C3 rates
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x > gpurun_out/pytest_f32p.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_f32p.log
for c in c5 c3; do timeout 600 python tools/f32_variant.py $c; done
