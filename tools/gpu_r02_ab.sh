#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baseline_steps.py tests/test_gpu_solver.py tests/test_gpu_kernels.py tests/test_gpu_api_ops.py tests/test_gpu_mixed_orders.py -m gpu -q -rf > gpurun_out/pytest_ab.log 2>&1
echo "pytest rc=$?"; tail -n 4 gpurun_out/pytest_ab.log
SF_GMRES_GRAPH=0 timeout 600 python tools/c2_step_ab.py 3 2>&1 | grep "^{"
timeout 600 python tools/step_timeline.py c2 20 10 gpurun_out/timeline_c2.json > gpurun_out/timeline_c2.log 2>&1
grep "steady\|block_solve\|fiber_rows\|end_wrench\|fiber_forces\|mgs" gpurun_out/timeline_c2.log | head -8
