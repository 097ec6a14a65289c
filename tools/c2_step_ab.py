"""Bench C2 state (bench.c2_step_state): per-step wall, GMRES wall and
matvec count, so the per-Arnoldi-step cost and the per-step setup separate.
Usage: SF_GMRES_GRAPH=0|1 python tools/c2_step_ab.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1602_05650_b200 import body, fiber, solver, system  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
st = bench.c2_step_state({"fiber": fiber, "body": body, "system": system})
params = solver.GmresParams(tolerance=1e-10)
orig = solver.gmres_solve
rec = {}


def timed_gmres(*a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = orig(*a, **k)
    torch.cuda.synchronize()
    rec["gmres_s"] = time.perf_counter() - t0
    return r


solver.gmres_solve = timed_gmres
for k in range(steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, info = solver.backward_euler_step(st, 1e-3, params, return_info=True)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    print(json.dumps({"graph": os.environ.get("SF_GMRES_GRAPH", "auto"), "step": k,
                      "step_ms": round(1e3 * el, 2), "gmres_ms": round(1e3 * rec["gmres_s"], 2),
                      "iters": info["iterations"], "matvecs": info["matvecs"],
                      "us_per_matvec_in_gmres": round(1e6 * rec["gmres_s"] / info["matvecs"], 1)}),
          flush=True)
