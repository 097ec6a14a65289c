"""Where does one GMRES iteration of a step go? (matvec, preconditioner, MGS)"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import _native, configs, solver  # noqa: E402
from paper_1602_05650_b200.system import InteractionCache  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
st = configs.aster(n_fibers=1024) if cfg == "c2" else configs.cloud_state(cfg)
dt = 1e-3 if cfg == "c2" else 5e-3


def timed(label, fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {1e3 * (time.perf_counter() - t0) / reps:9.3f} ms", flush=True)


t0 = time.perf_counter()
cache = InteractionCache(st)
torch.cuda.synchronize()
print(f"{'InteractionCache':40s} {1e3 * (time.perf_counter() - t0):9.3f} ms")
t0 = time.perf_counter()
op, rhs = solver.assemble_step_operator(st, dt, cache=cache)
torch.cuda.synchronize()
print(f"{'BlockOperator + rhs':40s} {1e3 * (time.perf_counter() - t0):9.3f} ms")
t0 = time.perf_counter()
prec = solver.Preconditioner(op)
torch.cuda.synchronize()
print(f"{'Preconditioner (LU)':40s} {1e3 * (time.perf_counter() - t0):9.3f} ms")
u = torch.randn(op.layout.size, dtype=torch.float64, device="cuda")
out = torch.empty_like(u)
timed("matvec (rows_device)", lambda: op.rows_device(u, False, out))
timed("  hi_apply only", lambda: cache.apply(op._f, op._densities(u), op._wr[:op.np] if op.np else None, out=op._ubar, check=False))
timed("  hi_apply + check_bad", lambda: cache.apply(op._f, op._densities(u), op._wr[:op.np] if op.np else None, out=op._ubar, check=True))
timed("preconditioner apply", lambda: prec.apply_device(u, out))
vec = solver._DeviceVectors(u.device)
h = torch.empty(1, dtype=torch.float64, device="cuda")
timed("dot", lambda: vec.dot_into(u, out, h))
timed("dot + axpy", lambda: (vec.dot_into(u, out, h), _native.call("sf_axpy_dev", h.data_ptr(), -1.0, 0, u.data_ptr(), out.data_ptr(), u.numel(), solver._stream())))
timed("host sync (item)", lambda: h.item())
params = solver.GmresParams(tolerance=1e-10)
t0 = time.perf_counter()
x, it, hist = solver.gmres_solve(op, prec, rhs, params)
torch.cuda.synchronize()
el = time.perf_counter() - t0
print(f"{'gmres_solve':40s} {1e3 * el:9.3f} ms  iters {it}  per iter {1e3 * el / it:.3f} ms")
