#!/bin/bash
for t in 1 2 4; do
  echo "tiles=$t"
  for c in c2 c4; do SF_SPLIT_TILES=$t timeout 300 python tools/matvec_profile.py $c | head -1; done
  SF_SPLIT_TILES=$t timeout 300 python tools/step_perf.py --config c1 --steps 4 | tail -1
  SF_SPLIT_TILES=$t timeout 300 python tools/pair_perf.py --config c5 --reps 1 --mode 3 2>/dev/null | tail -1
done
