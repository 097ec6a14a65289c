mkdir -p gpurun_out
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1; done
s=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo "bench20 rc=$? $(( $(date +%s) - s )) s"
python -c "
import json
d=json.loads(open('gpurun_out/bench20.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['variant_fp32c']['value'])"
s=$(date +%s); timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench20_ref.json 2> gpurun_out/bench20_ref.err; echo "ref20 rc=$? $(( $(date +%s) - s )) s"
tail -c 400 gpurun_out/bench20_ref.json
