#!/bin/bash
# symmetric-kernel unit-size sweep at C2 / C4-fiber sizes (whole evaluation, CUDA events)
for c in c2 c4; do
  for u in 256 384 512 640 768 1024; do
    SF_SYM_UNIT=$u timeout 300 python tools/sym_split_balance.py $c 8 --calibrate | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', $u, round(d['full_ms'],4))"
  done
done
