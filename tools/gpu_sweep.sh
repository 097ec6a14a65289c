timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in ${VARIANTS:-0 1 2 6 7}; do SF_PAIR_VARIANT=$v timeout 300 python tools/pair_perf.py --config c5 --reps 2 2>&1 | tail -1 | sed "s/^/v$v /"; done
