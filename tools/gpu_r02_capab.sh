#!/bin/bash
# capsule A/B in the same box: symmetric kernel and C2/C4 steps
for cap in 0 1; do
  echo "== SF_SYM_CAPSULE=$cap"
  for c in c2 c4; do SF_SYM_CAPSULE=$cap timeout 600 python tools/sym_split_balance.py $c 8 --calibrate; done
  SF_SYM_CAPSULE=$cap timeout 600 python tools/step_perf.py --config c2 --steps 3 | tail -2
  SF_SYM_CAPSULE=$cap timeout 900 python tools/step_perf.py --config c4 --steps 1 --tol 1e-8 | tail -1
done
