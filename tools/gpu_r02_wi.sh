#!/bin/bash
# warp-owns-i symmetric kernel: tests, kernel timing A/B at C2 (1024) and 2048 fibers, C2 step
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sym_kernels.py tests/test_gpu_sym_waves.py tests/test_gpu_sym_split.py tests/test_gpu_baseline_steps.py tests/test_gpu_system.py -m gpu -q -rf > gpurun_out/pytest_wi.log 2>&1
echo "pytest rc=$?"; tail -n 6 gpurun_out/pytest_wi.log
for wi in 0 1; do for nf in 1024 2048; do echo "wi=$wi nf=$nf"; SF_SYM_WI=$wi timeout 300 python tools/sym_aster_perf.py $nf 2>&1 | tail -n 1; done; done
SF_SYM_WI=1 timeout 600 python tools/c2_step_ab.py 3 2>&1 | grep "^{"
SF_SYM_WI=1 timeout 600 python tools/step_timeline.py c2 20 10 gpurun_out/timeline_c2_wi.json 2>&1 | grep "steady\|sym_task"
