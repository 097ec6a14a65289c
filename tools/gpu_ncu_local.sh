# HBM-bound batched local operators (self terms, fiber rows, block solves,
# near maps, partial reduce): duration and DRAM bytes per launch under ncu.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
K='regex:self_apply|block_solve|fiber_rows|fiber_forces|near_apply|sym_reduce|diag_div|end_wrench|wrench_reduce'
for c in c5 c3 c2; do
  timeout 600 python tools/matvec_profile.py $c > gpurun_out/plain_local_$c.log 2>&1 && \
  timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k "$K" --csv \
      python tools/matvec_profile.py $c > gpurun_out/ncu_local_$c.csv 2>&1
  echo "$c rc=$?"
done
