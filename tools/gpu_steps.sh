timeout 1200 python tools/step_perf.py --config c4 --steps 2 --tol 1e-8 2>&1 | tail -3
