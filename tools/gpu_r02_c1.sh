#!/bin/bash
# small-problem GMRES policy: C1 steps with graph / lag on and off
for g in 0 1; do for l in 0 1; do
  echo "== graph=$g lag=$l"
  SF_GMRES_GRAPH=$g SF_GMRES_LAG=$l timeout 300 python tools/step_perf.py --config c1 --steps 6 | tail -3
done; done
