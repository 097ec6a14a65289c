# full bench (both arms), smoke, launch list, and an ncu --set full of the FP32c kernel
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.json
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --step-config "" > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --step-config "" > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
timeout 300 python tools/pair_perf.py --config c5 --reps 1 --mode 1 > gpurun_out/plain_f32.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sym_task -c 1 \
    -o gpurun_out/prof_sym_f32_c5 python tools/pair_perf.py --config c5 --reps 1 --mode 1 > gpurun_out/ncu_f32.log 2>&1; echo "ncu f32 rc=$?"
