"""Rank balance of the multi-GPU symmetric fiber-pair split, measured on ONE
GPU: each rank's task share is run alone (sf_sbt_symmetric_tasks) and timed
with CUDA events; the max/mean ratio is the imbalance a world-size-W run
would see.  Compares the pair-count split with the modelled-cost split
(dist.cost_split of sf_sym_task_costs).  With --calibrate it also times the
whole evaluation once (run it with and without SF_SYM_NOFAST=1 to get the
checked-path cost ratio).
Usage: python tools/sym_split_balance.py c5|c2|c4 [world] [--calibrate]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_05650_b200 import _native, configs, dist  # noqa: E402
from paper_1602_05650_b200.operator import FiberHIOperator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
world = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 8
if cfg == "c2":
    st = configs.aster(n_fibers=1024)
    X = np.stack([f.X for f in st.fibers])
    eps = 1e-2
elif cfg == "c4":
    st = configs.confined_aster()
    X = np.stack([f.X for f in st.fibers])
    eps = 1e-2
else:
    cl = configs.make(cfg, seed=0)
    X, eps = cl.X, cl.eps
dev = torch.device("cuda")
op = FiberHIOperator(X, eps, device=dev, shard=(0, world))
f = torch.as_tensor(np.random.default_rng(1).standard_normal(X.shape), device=dev).reshape(-1, 3)
out = torch.empty((op.N, 3), dtype=torch.float64, device=dev)
lib = _native.load()
res = {"config": cfg, "world": world, "N": op.N}


def time_range(t0, cnt, reps=2):
    _native.call("sf_sbt_symmetric_tasks", op.X.data_ptr(), op.groups.data_ptr(), op.N, op.n,
                 f.data_ptr(), op.wnode.data_ptr(), op.dcoef.data_ptr(), op.pref, op.mode, t0, cnt,
                 out.data_ptr(), op.bad.data_ptr(), None)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        _native.call("sf_sbt_symmetric_tasks", op.X.data_ptr(), op.groups.data_ptr(), op.N, op.n,
                     f.data_ptr(), op.wnode.data_ptr(), op.dcoef.data_ptr(), op.pref, op.mode, t0,
                     cnt, out.data_ptr(), op.bad.data_ptr(), None)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


if "--calibrate" in sys.argv:
    T = int(lib.sf_sym_task_count(op.N, op.n, op.mode))
    res["nofast"] = os.environ.get("SF_SYM_NOFAST", "0")
    res["full_ms"] = time_range(0, T)
else:
    costs = dist.sym_task_costs(op.X.reshape(-1, 3), op.groups, op.N, op.n, op.mode)
    for name, split in (("pairs", dist.pair_split(op.N, op.n, op.mode, world)),
                        ("cost", dist.cost_split(costs, world))):
        ms = [time_range(t0, cnt) for t0, cnt in split]
        model = [float(costs[t0:t0 + cnt].sum()) for t0, cnt in split]
        res[name] = {"ranges": split, "ms": ms, "imbalance": max(ms) / np.mean(ms) - 1.0,
                     "model_imbalance": max(model) / np.mean(model) - 1.0}
print(json.dumps(res), flush=True)
