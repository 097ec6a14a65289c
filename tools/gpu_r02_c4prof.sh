#!/bin/bash
# refreshed C4 launch lists: one block-operator matvec + preconditioner, and
# three Arnoldi steps of a C4 solve
mkdir -p gpurun_out
timeout 600 python tools/matvec_profile.py c4 > gpurun_out/plain_c4.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/matvec_profile.py c4 > gpurun_out/ncu_matvec_c4.csv 2>&1; echo "c4 matvec rc=$?"
cat gpurun_out/plain_c4.log | tail -1
timeout 900 python tools/gmres_iter_profile.py c4 20 3 > gpurun_out/iter_c4.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/gmres_iter_profile.py c4 20 3 > gpurun_out/ncu_iter_c4.csv 2>&1; echo "c4 iter rc=$?"
tail -1 gpurun_out/iter_c4.log
