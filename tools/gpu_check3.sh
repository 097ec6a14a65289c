mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py tests/test_gpu_cross.py tests/test_gpu_solver.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/step_breakdown.py c2 2>&1 | grep -v Interaction | tail -12
timeout 300 python tools/matvec_profile.py c4 2>&1 | head -2
timeout 300 python tools/pair_perf.py --config c5 --reps 3 --mode 0 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/c2_matvec_launches.csv python tools/matvec_profile.py c2 > /dev/null 2>&1; echo ncu rc=$?
