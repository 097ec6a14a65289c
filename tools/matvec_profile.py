"""One block-operator matvec + preconditioner apply inside a
cudaProfilerStart/Stop window, for `ncu --profile-from-start off` launch lists.
Usage: python tools/matvec_profile.py c2|c4|c3|c3_scaled"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
st = {"c2": lambda: configs.aster(n_fibers=1024), "c4": lambda: configs.confined_aster()}.get(
    cfg, lambda: configs.cloud_state(cfg))()
dt = 1e-3 if cfg in ("c2", "c4") else 5e-3
op, rhs = solver.assemble_step_operator(st, dt)
prec = solver.Preconditioner(op)
u = torch.randn(op.layout.size, dtype=torch.float64, device="cuda")
out = torch.empty_like(u)
for _ in range(3):
    prec.apply_device(op.rows_device(u, False, out))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    prec.apply_device(op.rows_device(u, False, out))
torch.cuda.synchronize()
print(f"matvec+prec {1e3 * (time.perf_counter() - t0) / 10:.3f} ms", flush=True)
torch.cuda.profiler.start()
prec.apply_device(op.rows_device(u, False, out))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
