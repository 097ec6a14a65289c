"""Experiment: GMRES iterations on the C2 aster with the reference's block-Jacobi
preconditioner vs one that also couples the particle block to the fibers
(particle rows x all columns + fiber rows x the particle's U, Omega columns,
solved by a Schur complement).  Prototype built from operator probes; not a
product path."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
st = configs.aster(n_fibers=nf)
op, rhs = solver.assemble_step_operator(st, 1e-3)
prec = solver.Preconditioner(op)
lay = op.layout
n = lay.size
nb = lay.fib_off                       # particle unknowns [U Omega q1]
dev = op.device
f64 = dict(dtype=torch.float64, device=dev)
params = solver.GmresParams(tolerance=1e-10, max_iterations=2000)
rhs_d = torch.as_tensor(rhs, **f64) if not torch.is_tensor(rhs) else rhs

t0 = time.perf_counter()
_, it_ref, _ = solver.gmres_solve(op, prec, rhs_d, params)
torch.cuda.synchronize()
print(f"block-Jacobi (reference): {it_ref} iterations, {time.perf_counter() - t0:.2f} s", flush=True)


def A(u):
    return op.rows_device(u, False).clone()


t0 = time.perf_counter()
Abb = torch.empty((nb, nb), **f64)
Afb6 = torch.empty((n - nb, 6), **f64)
e = torch.zeros(n, **f64)
for j in range(nb):
    e[j] = 1.0
    col = A(e)
    e[j] = 0.0
    Abb[:, j] = col[:nb]
    if j < 6:
        Afb6[:, j] = col[nb:]
torch.cuda.synchronize()
print(f"probed particle block {nb}x{nb}: {time.perf_counter() - t0:.1f} s", flush=True)


def Dinv(vf):
    v = torch.zeros(n, **f64)
    v[nb:] = vf
    return prec.apply_device(v)[nb:].clone()


def Abf(yf):
    u = torch.zeros(n, **f64)
    u[nb:] = yf
    return A(u)[:nb]


W = torch.stack([Dinv(Afb6[:, j]) for j in range(6)], dim=1)
S = Abb.clone()
S[:, :6] -= torch.stack([Abf(W[:, j]) for j in range(6)], dim=1)
LU, piv = torch.linalg.lu_factor(S)


class Coupled:
    def apply_device(self, v, out=None):
        yf = Dinv(v[nb:])
        zb = torch.linalg.lu_solve(LU, piv, (v[:nb] - Abf(yf))[:, None])[:, 0]
        z = torch.empty(n, **f64) if out is None else out
        z[:nb] = zb
        z[nb:] = yf - W @ zb[:6]
        return z

    apply = apply_device


t0 = time.perf_counter()
x2, it2, _ = solver.gmres_solve(op, Coupled(), rhs_d, params)
torch.cuda.synchronize()
print(f"particle-coupled: {it2} iterations, {time.perf_counter() - t0:.2f} s", flush=True)
x1, _, _ = solver.gmres_solve(op, prec, rhs_d, params)


def rel(a, b):
    return float((a - b).norm() / b.norm())


for name, x in (("block-Jacobi", x1), ("coupled", x2)):
    print(f"{name}: true residual |b - A x| / |b| = {rel(A(x), rhs_d):.3e}")
import numpy as np  # noqa: E402
xs = torch.as_tensor(np.concatenate([np.arange(s_.start, s_.stop) for s_ in lay.X]), device=dev)
ts = torch.as_tensor(np.concatenate([np.arange(s_.start, s_.stop) for s_ in lay.T]), device=dev)
print("rel diff, fiber X", rel(x2[xs], x1[xs]), " T", rel(x2[ts], x1[ts]))
print("rel diff, U Omega", rel(x2[:6], x1[:6]), "q1", rel(x2[6:nb], x1[6:nb]))
# a tighter reference solve for the forward error
xt, itt, _ = solver.gmres_solve(op, prec, rhs_d, solver.GmresParams(tolerance=1e-12, max_iterations=3000))
print(f"tight block-Jacobi solve (1e-12): {itt} it, true residual {rel(A(xt), rhs_d):.2e}")
for name, x in (("block-Jacobi", x1), ("coupled", x2)):
    print(f"  {name} error vs tight: X {rel(x[xs], xt[xs]):.2e} T {rel(x[ts], xt[ts]):.2e} "
          f"particle {rel(x[:nb], xt[:nb]):.2e}")
x3, it3, _ = solver.gmres_solve(op, Coupled(), rhs_d, solver.GmresParams(tolerance=1e-12, max_iterations=3000))
print(f"coupled at 1e-12: {it3} it; error vs tight: X {rel(x3[xs], xt[xs]):.2e} T {rel(x3[ts], xt[ts]):.2e}")
