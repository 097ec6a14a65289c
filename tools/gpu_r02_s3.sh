#!/bin/bash
# session-3 re-entry check: full GPU suite, smoke, both bench arms as the driver runs them
mkdir -p gpurun_out
s=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS} > gpurun_out/pytest.log 2>&1
echo "pytest rc=$? $(( $(date +%s) - s )) s"; tail -n 15 gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
s=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? $(( $(date +%s) - s )) s"
tail -c 600 gpurun_out/bench.json
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? $(( $(date +%s) - s )) s"
