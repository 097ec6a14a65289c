#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_dist_solver.py tests/test_gpu_fp32c_krylov.py -m gpu -q -rf > gpurun_out/pytest_misc.log 2>&1
echo "pytest rc=$?"; tail -n 12 gpurun_out/pytest_misc.log
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variant --step-config c1,c2,c2:body > gpurun_out/bench_steps.json 2> gpurun_out/bench_steps.err
echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/bench_steps.json').read().strip().splitlines()[-1])
for s in d['implicit_steps']: print(s['config'][:30], s['preconditioner'][:12], round(s['ms_per_step'],1), s['gmres_iterations'])"
timeout 900 python tools/tree_crossover.py 512 2048 4096 16384 > gpurun_out/tree_crossover.log 2>&1; echo "tree rc=$?"; cat gpurun_out/tree_crossover.log | tail -5
