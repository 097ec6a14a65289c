#!/bin/bash
# FP32c kernel variants at C5 (scalar FFMA vs packed FFMA2) and the recalibrated rank split
mkdir -p gpurun_out
for v in 34 134 124 136; do
  SF_SYM_F32_VARIANT=$v timeout 600 python tools/f32_variant.py c5 >> gpurun_out/f32_variants.log 2>&1
done
cat gpurun_out/f32_variants.log
for c in c4 c2 c5; do
  timeout 900 python tools/sym_split_balance.py $c 8 > gpurun_out/split2_$c.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/split2_$c.json').read().strip().splitlines()[-1])
for k in ('pairs','cost'): print('$c', k, 'imbalance %.4f model %.4f' % (d[k]['imbalance'], d[k]['model_imbalance']))"
done
