#!/bin/bash
# full GPU suite + implicit-step bench lines
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?"; tail -n 8 gpurun_out/pytest_full.log
timeout 1500 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variant --step-config c1,c2,c2:body,c4,c4:body > gpurun_out/bench_steps.json 2> gpurun_out/bench_steps.err
echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_steps.json').read().strip().splitlines()[-1])
for s in d['implicit_steps']: print(s['config'][:30], s['preconditioner'][:12], round(s['ms_per_step'],1), s['gmres_iterations'])"
