"""Setup cost of one implicit step (cache, operator, preconditioner) on C2/C4,
warm, with SF_DEBUG_TIMING laps of the InteractionCache."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402
from paper_1602_05650_b200.system import InteractionCache  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
st = configs.aster(n_fibers=1024) if cfg == "c2" else configs.confined_aster()
for rep in range(2):
    if rep == 1:
        os.environ["SF_DEBUG_TIMING"] = "1"
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cache = InteractionCache(st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    op, rhs = solver.assemble_step_operator(st, 1e-3, cache=cache)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    prec = solver.Preconditioner(op, body_coupling=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{cfg} rep {rep}: cache {1e3*(t1-t0):.1f} ms, operator+rhs {1e3*(t2-t1):.1f} ms, "
          f"preconditioner {1e3*(t3-t2):.1f} ms", flush=True)
