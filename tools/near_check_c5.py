"""Diagnostic: near-field pairs of the C5 cloud under the reference's near
criterion (InteractionCache) vs the bench operator's map, and the difference
of the two non-local outputs."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, system  # noqa: E402
from paper_1602_05650_b200.fiber import Fiber  # noqa: E402
from paper_1602_05650_b200.operator import FiberHIOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cloud = configs.make(name, seed=0)
f = configs.forces(cloud, seed=1)
st = system.SystemState([Fiber(X, eps=cloud.eps, E=cloud.E) for X in cloud.X])
cache = system.InteractionCache(st)
print("near fiber pairs (reference criterion):", len(cache.near_fiber), "rows", cache.near_nrows)
res = system.complementary_velocities(st, fiber_forces=list(f), cache=cache)
ua = np.concatenate(res.fibers)
op = FiberHIOperator(cloud.X, cloud.eps)
ub = op.apply(torch.as_tensor(f, device="cuda"), self_terms=False)[0].cpu().numpy()
d = np.linalg.norm(ua - ub, axis=1)
print("rel L2 diff", np.linalg.norm(ua - ub) / np.linalg.norm(ua), "rows differing > 1e-10:",
      int((d > 1e-10 * np.abs(ua).max()).sum()))
if len(cache.near_fiber):
    t = sorted({t for t, _, _ in cache.near_fiber})
    print("first near targets", t[:10])
    near = [(t, l, W.cpu().numpy() if torch.is_tensor(W) else W) for t, l, W in cache.near_fiber]
    op2 = FiberHIOperator(cloud.X, cloud.eps, near=near)
    uc = op2.apply(torch.as_tensor(f, device="cuda"), self_terms=False)[0].cpu().numpy()
    print("with the cache's near maps: rel L2 diff", np.linalg.norm(ua - uc) / np.linalg.norm(ua))
