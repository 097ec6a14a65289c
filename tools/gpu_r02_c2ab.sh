#!/bin/bash
# C2 per-step A/B: default, unit 512, forced cross kernel, both
for cfg in "" "SF_SYM_UNIT=512" "SF_CROSS=2" "SF_SYM_UNIT=512 SF_CROSS=2"; do
  echo "== $cfg"
  env $cfg timeout 600 python tools/step_perf.py --config c2 --steps 3 | tail -2
done
