# SF_SYM_UNIT sweep of the symmetric kernel at mid sizes (tools/pair_perf.py)
for fib in 512 1024 4096; do
  for u in default 256 384 512 640 768 1024 1536 2048; do
    if [ $u = default ]; then
      r=$(timeout 120 python tools/pair_perf.py --config c3_scaled --fibers $fib --reps 5 2>&1 | tail -1)
    else
      r=$(SF_SYM_UNIT=$u timeout 120 python tools/pair_perf.py --config c3_scaled --fibers $fib --reps 5 2>&1 | tail -1)
    fi
    echo "fibers=$fib unit=$u $r"
  done
done
