#!/bin/bash
# both bench arms as the driver runs them (timed), then smoke
mkdir -p gpurun_out
s=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? $(( $(date +%s) - s )) s"
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$? $(( $(date +%s) - s )) s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
