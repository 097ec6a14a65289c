"""FP32-compute / FP64-accumulate fiber pair sums on the inputs GMRES
actually feeds the operator, at full BASELINE size (north_star: rel L2
<= 1e-5 of the FP64 operator).

The i.i.d. N(0,1) forces of the headline check are smooth in the sense that
matters: every slab of sources carries a net force, so no cancellation.
Inside a solve the operator sees elastic force densities -E D_s^4 X +
D_s(T X_s) of the Krylov vectors and of perturbed centrelines; per fiber
these are nearly self-balanced, so their far field is a cancellation of
large terms.  These tests apply both precisions to such inputs:

* the elastic force density of the perturbed C3 / C5 centrelines (T = 0);
* the force densities of the first Krylov vectors of a C3 step,
  w_1 = M A b / |.|, w_2 = M A w_1 / |.| (b = M rhs): the span GMRES builds,
  through the step's own fiber-force kernel (sf_fiber_forces)."""

import ctypes

import numpy as np
import pytest
import torch

from paper_1602_05650_b200 import _native, configs, solver
from paper_1602_05650_b200.system import InteractionCache

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _forces(op, u):
    """Fiber force densities (N, 3) of the unknown vector u (sf_fiber_forces)."""
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f = torch.empty_like(op._f)
    for b in op.batches:
        _native.call("sf_fiber_forces", ctypes.byref(b.sys), u.data_ptr(), 0, f.data_ptr(), st)
    return f


def _both(state, f):
    """Fiber-target velocities of the fiber forces f in FP64 and FP32c."""
    out = []
    for mode in (_native.SF_MODE_FP64, _native.SF_MODE_FP32C):
        c = InteractionCache(state, mode=mode)
        u = c.apply(f, None, None, check=True)[c.fiber_slice]
        out.append(u.clone())
    return out


def _rel(a, b):
    return float((a - b).norm() / b.norm())


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_fp32c_on_elastic_forces_of_perturbed_fibers(cuda, cfg):
    st = configs.cloud_state(cfg, seed=0)
    op = solver.BlockOperator(st, 5e-3)
    u = torch.zeros(op.layout.size, dtype=torch.float64, device=cuda)
    X = torch.as_tensor(np.stack([f.X for f in st.fibers]), device=cuda)
    n = op.n
    idx = torch.arange(op.nf, device=cuda)[:, None] * (4 * n) + op.layout.fib_off
    u.view(-1)[(idx + torch.arange(3 * n, device=cuda)[None, :]).reshape(-1)] = X.reshape(-1)
    f = _forces(op, u)
    fn = f.view(op.nf, n, 3)            # per fiber net force vs force scale
    balance = float(fn.sum(dim=1).norm() / fn.abs().sum(dim=1).norm())
    a64, a32 = _both(st, f)
    err = _rel(a32, a64)
    print(f"{cfg} elastic-force inputs (net/abs {balance:.2e}): FP32c rel L2 {err:.2e}")
    assert err <= TOL, err


def test_fp32c_on_krylov_vectors_of_a_c3_step(cuda):
    st = configs.cloud_state("c3", seed=0)
    op, rhs = solver.assemble_step_operator(st, 5e-3)
    prec = solver.Preconditioner(op)
    b = prec.apply_device(rhs)
    w = b / b.norm()
    errs = []
    for k in range(3):
        f = _forces(op, w)
        a64, a32 = _both(st, f)
        errs.append(_rel(a32, a64))
        w = prec.apply_device(op.rows_device(w, False))
        w = w / w.norm()
    print("C3 Krylov inputs: FP32c rel L2", ["%.2e" % e for e in errs])
    assert max(errs) <= TOL, errs
