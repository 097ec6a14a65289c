#!/bin/bash
# round-2 check: GPU tests, then the C5 matvec with the wave budgets
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 30 gpurun_out/pytest.log
for mb in 192 96 384; do
  SF_SYM_WAVE_MB=$mb timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-variant \
     --step-config '' > gpurun_out/bench_mb$mb.json 2> gpurun_out/bench_mb$mb.err
  echo "mb=$mb rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_mb$mb.json').read().strip().splitlines()[-1]);print(d['value']/1e9, d['roofline']['frac'], d['ms_per_step'], d['gpu_launches'])"
done
SF_SYM_STREAMS=1 timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-variant --step-config '' > gpurun_out/bench_s1.json 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/bench_s1.json').read().strip().splitlines()[-1]);print('streams1', d['value']/1e9, d['roofline']['frac'])"
