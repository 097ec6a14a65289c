timeout 900 python tools/step_perf.py --config c3_scaled --steps 2 2>&1 | tail -3
timeout 900 python tools/step_perf.py --config c3 --steps 2 2>&1 | tail -3
