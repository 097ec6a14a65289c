"""Launch list of GMRES iterations of one implicit step: the profiler window
(cudaProfilerStart/Stop, for `ncu --profile-from-start off`) opens at the
START-th matvec and closes COUNT matvecs later, so it holds COUNT whole
Arnoldi steps (matvec, preconditioner, fused MGS, Givens, status copy).
Usage: python tools/gmres_iter_profile.py c2|c4|c3 [START] [COUNT]"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
start = int(sys.argv[2]) if len(sys.argv) > 2 else 20
count = int(sys.argv[3]) if len(sys.argv) > 3 else 3
st = {"c2": lambda: configs.aster(n_fibers=1024), "c4": lambda: configs.confined_aster()}.get(
    cfg, lambda: configs.cloud_state(cfg))()
dt = 1e-3 if cfg in ("c2", "c4") else 5e-3
params = solver.GmresParams(tolerance=1e-8 if cfg == "c4" else 1e-10)
os.environ["SF_GMRES_GRAPH"] = "0"      # launch by launch: the profiler window counts matvec calls
st, info = solver.backward_euler_step(st, dt, params, return_info=True)      # warm-up step
orig = solver.BlockOperator.rows_device
calls = [0]


def rows(self, u, constants, out=None):
    if not constants:
        calls[0] += 1
        if calls[0] == start:
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        elif calls[0] == start + count:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
    return orig(self, u, constants, out)


solver.BlockOperator.rows_device = rows
torch.cuda.synchronize()
t0 = time.perf_counter()
st, info = solver.backward_euler_step(st, dt, params, return_info=True)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(f"{cfg}: step {1e3 * el:.1f} ms, {info['iterations']} iterations, {info['matvecs']} matvecs, "
      f"{1e3 * el / info['matvecs']:.3f} ms per matvec", flush=True)
