#!/bin/bash
# CUDA-graph Arnoldi step: GPU tests, C2 step timings graph on/off, unit-size sweep
mkdir -p gpurun_out
timeout 1500 python -m pytest ${PYTEST_TARGETS:-tests} -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 15 gpurun_out/pytest.log
for g in 0 1; do
  SF_GMRES_GRAPH=$g timeout 600 python tools/step_perf.py --config c2 --steps 3 > gpurun_out/c2_graph$g.log 2>&1
  echo "graph=$g rc=$?"; tail -3 gpurun_out/c2_graph$g.log
done
for u in 512 1024; do
  SF_SYM_UNIT=$u timeout 600 python tools/step_perf.py --config c2 --steps 2 > gpurun_out/c2_unit$u.log 2>&1
  echo "unit=$u rc=$?"; tail -2 gpurun_out/c2_unit$u.log
done
