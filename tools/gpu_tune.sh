set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for tb in 1 2 4; do SF_PAIR_TB=$tb timeout 300 python tools/pair_perf.py --config c5 2>&1 | tail -1; done
SF_PAIR_TB=2 timeout 300 python tools/pair_perf.py --config c5 --mode 1 2>&1 | tail -1
