#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sym_waves.py -m gpu -q -rf 2>&1 | tail -3
timeout 600 python tools/gmres_iter_profile.py c2 20 3 > gpurun_out/iter_c2.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/gmres_iter_profile.py c2 20 3 > gpurun_out/ncu_iter_c2.csv 2>&1; echo "c2 iter rc=$?"
tail -1 gpurun_out/iter_c2.log
