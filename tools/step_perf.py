"""Implicit-step timing on a config (helper; the bench reports the headline)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--fibers", type=int, default=0)
ap.add_argument("--tol", type=float, default=1e-10)
a = ap.parse_args()
if not a.fibers:
    a.fibers = 2048 if a.config == "c4" else 1024
if a.config == "c1":
    import bench
    from paper_1602_05650_b200 import body, fiber, system
    st = bench.c1_step_state({"fiber": fiber, "body": body, "system": system})
    dt = 5e-3
elif a.config == "c2":
    st = configs.aster(n_fibers=a.fibers)
    dt = 1e-3
elif a.config == "c4":
    st = configs.confined_aster(n_fibers=a.fibers)
    dt = 1e-3
else:
    st = configs.cloud_state(a.config)
    dt = 5e-3
params = solver.GmresParams(tolerance=a.tol)
for k in range(a.steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, info = solver.backward_euler_step(st, dt, params, return_info=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    info["near"] = info.get("near")
    print(json.dumps({"config": a.config, "step": k, "s": el, "iters": info["iterations"],
                      "matvecs": info["matvecs"], "dt": info["dt"]}), flush=True)
