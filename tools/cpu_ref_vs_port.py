"""Reference pair sums on the box's host cores: slenderflow's own numba
kernels vs the oracle's C port, same C5 row sample (bench.cpu_pair_rate)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
from oracle import pairs  # noqa: E402
from paper_1602_05650_b200 import configs  # noqa: E402

cl = configs.make("c5", seed=0)
f = configs.forces(cl, seed=1)
pairs.set_num_threads(bench.host_threads())
for use_ref in (True, False, True, False):
    r, dt, n, th, kind = bench.cpu_pair_rate(cl.X, f, cl.eps, 2000, seed=3, use_reference=use_ref)
    print(json.dumps({"kind": kind, "pairs_per_s": r, "seconds": dt, "threads": th}), flush=True)
