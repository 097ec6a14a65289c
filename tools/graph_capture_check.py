"""Does the GMRES Arnoldi-step graph capture succeed for a config?  Runs two
implicit steps with SF_GMRES_GRAPH=1 and reports capture failures (with
their traceback) and the step times.  Usage: python tools/graph_capture_check.py c1|c2|c4"""
import logging
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
os.environ["SF_GMRES_GRAPH"] = "1"
os.environ.setdefault("SF_GMRES_CAPTURE_TRACE", "1")
logging.basicConfig(level=logging.WARNING)
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
st = {"c2": lambda: configs.aster(n_fibers=1024), "c4": lambda: configs.confined_aster(),
      "c1": lambda: configs.cloud_state("c1")}.get(cfg, lambda: configs.cloud_state(cfg))()
dt = 1e-3 if cfg in ("c2", "c4") else 5e-3
params = solver.GmresParams(tolerance=1e-8 if cfg == "c4" else 1e-10)
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, info = solver.backward_euler_step(st, dt, params, return_info=True)
    torch.cuda.synchronize()
    print(f"{cfg} step {k}: {1e3 * (time.perf_counter() - t0):.2f} ms, {info['iterations']} its",
          flush=True)
