#!/bin/bash
# capsule slab bounds: correctness, then symmetric-kernel and C2 step timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -x --deselect tests/test_gpu_baseline_steps.py > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 8 gpurun_out/pytest.log
for c in c2 c4 c5; do timeout 600 python tools/sym_split_balance.py $c 8 --calibrate; done
SF_SYM_F32_VARIANT=34 timeout 600 python tools/f32_variant.py c5
timeout 600 python tools/step_perf.py --config c2 --steps 3 | tail -2
timeout 900 python tools/step_perf.py --config c4 --steps 1 | tail -1
