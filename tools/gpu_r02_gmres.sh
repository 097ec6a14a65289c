#!/bin/bash
# device-Givens GMRES: GPU tests, then C2 step timings with lag 0 / 1
mkdir -p gpurun_out
timeout 1500 python -m pytest ${PYTEST_TARGETS:-tests} -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 25 gpurun_out/pytest.log
for lag in 0 1; do
  SF_GMRES_LAG=$lag timeout 600 python tools/step_perf.py --config c2 --steps 3 > gpurun_out/c2_lag$lag.log 2>&1
  echo "lag=$lag rc=$?"; cat gpurun_out/c2_lag$lag.log | tail -3
done
