for v in 224 124 233 223 232; do
  SF_SYM_VARIANT=$v timeout 120 python tools/sym_aster_perf.py 1024 2>&1 | tail -1
done
for m in 128 384 512; do
  SF_SYM_UNIT=$m timeout 120 python tools/sym_aster_perf.py 1024 2>&1 | tail -1
done
timeout 120 python tools/sym_aster_perf.py 2048 2>&1 | tail -1
