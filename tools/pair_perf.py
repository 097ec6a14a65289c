"""Time the fused pair kernel on a config (tuning helper; not the bench)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, kernels  # noqa: E402
from paper_1602_05650_b200.operator import FiberHIOperator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--fibers", type=int, default=0)
a = ap.parse_args()
kw = {"n_fibers": a.fibers} if a.fibers else {}
cloud = configs.make(a.config, seed=0, **kw)
f = torch.as_tensor(configs.forces(cloud), device="cuda")
op = FiberHIOperator(cloud.X, cloud.eps, mode=a.mode)
u = torch.empty((op.N, 3), dtype=torch.float64, device="cuda")
op.apply(f, out_nl=u, self_terms=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    op.apply(f, out_nl=u, self_terms=False)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.reps
peak, _ = kernels.dfma_peak(1 << 15)
tf = op.pairs_per_apply * 35 / (ms * 1e-3) / 1e12
print(json.dumps({"config": a.config, "tb": os.environ.get("SF_PAIR_TB", "2"), "mode": a.mode,
                  "ms": ms, "gpairs_s": op.pairs_per_apply / (ms * 1e-3) / 1e9, "tflops": tf,
                  "peak_tflops": peak / 1e12, "frac": tf * 1e12 / peak}))
