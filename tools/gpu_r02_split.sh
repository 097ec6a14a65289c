#!/bin/bash
# cost-balanced rank split: tests, one-GPU share timings, checked-path calibration
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sym_split.py tests/test_gpu_kernels.py tests/test_gpu_dist_solver.py tests/test_gpu_bench_multirank.py -m gpu -q -rf > gpurun_out/pytest_split.log 2>&1
echo "pytest rc=$?"; tail -n 15 gpurun_out/pytest_split.log
for nf in 0 1; do
  SF_SYM_NOFAST=$nf timeout 600 python tools/sym_split_balance.py c5 8 --calibrate >> gpurun_out/split_cal.log 2>&1
  SF_SYM_NOFAST=$nf timeout 600 python tools/sym_split_balance.py c2 8 --calibrate >> gpurun_out/split_cal.log 2>&1
done
cat gpurun_out/split_cal.log
for c in c2 c5 c4; do
  timeout 900 python tools/sym_split_balance.py $c 8 > gpurun_out/split_$c.json 2>&1
  echo "$c rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/split_$c.json').read().strip().splitlines()[-1])
for k in ('pairs','cost'): print('$c', k, 'imbalance %.4f model %.4f' % (d[k]['imbalance'], d[k]['model_imbalance']), ['%.1f' % x for x in d[k]['ms']])"
done
