#!/bin/bash
# round-2 check: failing GPU tests, the per-block operator diagnostic, then the
# C5 matvec with the wave budgets
mkdir -p gpurun_out
timeout 1200 python -m pytest ${PYTEST_TARGETS:-tests} -m gpu -q -rf -x ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 30 gpurun_out/pytest.log
timeout 600 python tools/tension_diag.py bstep_c1.npz bstep_aster256.npz > gpurun_out/tension.log 2>&1
echo "diag rc=$?"; cat gpurun_out/tension.log | tail -20
for mb in 192 96 384; do
  SF_SYM_WAVE_MB=$mb timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-variant \
     --step-config '' > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err
  echo "mb=$mb rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_mb$mb.json').read().strip().splitlines()[-1]);print(d['value']/1e9, d['roofline']['frac'], d['ms_per_step'], d['gpu_launches'])"
done
