set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
make -s -C oracle
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 300 python -c "from paper_1602_05650_b200 import kernels; print('dfma', kernels.dfma_peak(1<<16)); print('dfma', kernels.dfma_peak(1<<17))" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/bench1.log
