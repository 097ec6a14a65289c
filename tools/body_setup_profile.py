"""Where does the body-coupled preconditioner's setup and apply go? (C2 / C4)"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
st = configs.aster(n_fibers=1024) if cfg == "c2" else configs.confined_aster()
op, rhs = solver.assemble_step_operator(st, 1e-3)


def timed(label, fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{cfg} {label:44s} {1e3 * (time.perf_counter() - t0) / reps:8.2f} ms", flush=True)
    return r


p0 = timed("block-Jacobi setup", lambda: solver.Preconditioner(op))
p1 = timed("coupled setup (cold particle inverse)", lambda: solver.Preconditioner(op, body_coupling=True))
p1 = timed("coupled setup (cached particle inverse)", lambda: solver.Preconditioner(op, body_coupling=True), 3)
v = torch.randn(op.layout.size, dtype=torch.float64, device=op.device)
timed("apply block-Jacobi", lambda: p0.apply_device(v), 20)
timed("apply coupled", lambda: p1.apply_device(v), 20)
y = torch.zeros(op.layout.size, dtype=torch.float64, device=op.device)
timed("particle_rows_device", lambda: op.particle_rows_device(y), 20)
timed("matvec", lambda: op.rows_device(v, False), 10)
x, it, _ = timed("gmres (coupled)", lambda: solver.gmres_solve(op, p1, rhs, solver.GmresParams(tolerance=1e-10)))
print("iterations", it)
timed("full step (coupled)", lambda: solver.backward_euler_step(st, 1e-3, solver.GmresParams(tolerance=1e-10), body_coupling=True), 3)
cp = p1.coupled
if cp is not None:
    r = torch.randn(cp["pend"], dtype=torch.float64, device=op.device)
    timed("  GEMV S^-1 (pend x pend)", lambda: torch.mv(cp["Sinv"], r), 50)
    zc = torch.randn(cp["W"].shape[1], dtype=torch.float64, device=op.device)
    tgt = torch.zeros(cp["W"].shape[0], dtype=torch.float64, device=op.device)
    timed("  addmv W (fiber unknowns x 6)", lambda: tgt.addmv_(cp["W"], zc, alpha=-1.0), 50)
    timed("  block-Jacobi only", lambda: p1._block_jacobi(v), 50)
