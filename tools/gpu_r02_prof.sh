#!/bin/bash
# per-iteration launch lists of the C2 / C4 GMRES loop
mkdir -p gpurun_out
for c in c2 c4; do
  timeout 600 python tools/gmres_iter_profile.py $c 20 3 > gpurun_out/iter_$c.log 2>&1
  echo "$c plain rc=$?"; cat gpurun_out/iter_$c.log | tail -2
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      python tools/gmres_iter_profile.py $c 20 3 > gpurun_out/ncu_iter_$c.csv 2>&1
  echo "$c ncu rc=$?"
done
