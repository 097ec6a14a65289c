#!/bin/bash
# round-2 evidence: both bench arms as the driver runs them, the launch list of
# the same command, and one full ncu capture of the dominant kernel
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/bench.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -c 600 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-variant --step-config "" > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 300 python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/plain_sym.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sym_task -c 1 \
    -o gpurun_out/prof_sym_c5 python tools/pair_perf.py --config c5 --reps 1 > gpurun_out/ncu_sym.log 2>&1
echo "ncu full rc=$?"; tail -2 gpurun_out/ncu_sym.log
