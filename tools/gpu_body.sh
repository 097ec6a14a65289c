mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_body_coupling.py tests/test_gpu_solver.py -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variant --step-config c2,c2:body,c4,c4:body 2>gpurun_out/body_bench.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for s in d['implicit_steps']: print({k: s.get(k) for k in ('config','preconditioner','ms_per_step','gmres_iterations','error')})
"
tail -3 gpurun_out/body_bench.err
