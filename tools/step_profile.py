"""Steady-state phase timing of implicit steps (second step onwards)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402
from paper_1602_05650_b200.system import InteractionCache  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
st = {"c2": lambda: configs.aster(n_fibers=1024), "c4": lambda: configs.confined_aster()}.get(
    cfg, lambda: configs.cloud_state(cfg))()
dt = 1e-3 if cfg in ("c2", "c4") else 5e-3
tol = 1e-8 if cfg == "c4" else 1e-10
params = solver.GmresParams(tolerance=tol)
if os.environ.get("STEP_WARMUP", "1") != "0":
    solver.backward_euler_step(st, dt, params)   # warm-up


def lap(t0, label):
    torch.cuda.synchronize()
    t = time.perf_counter()
    print(f"{label:28s} {1e3 * (t - t0):9.2f} ms", flush=True)
    return t


for rep in range(int(os.environ.get("STEP_REPS", "2"))):
    t = time.perf_counter()
    cache = InteractionCache(st)
    t = lap(t, "InteractionCache")
    op, rhs = solver.assemble_step_operator(st, dt, cache=cache)
    t = lap(t, "BlockOperator + rhs")
    prec = solver.Preconditioner(op)
    t = lap(t, "Preconditioner")
    x, it, hist = solver.gmres_solve(op, prec, rhs, params)
    t2 = lap(t, f"GMRES ({it} it)")
    print(f"{'  per iteration':28s} {1e3 * (t2 - t) / it:9.2f} ms")
    print("---")
