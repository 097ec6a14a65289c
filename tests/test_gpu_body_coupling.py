"""Body-coupled preconditioner (not in the reference; opt-in): its pieces are
checked against the operator itself, and steps taken with it reproduce the
reference's golden positions (<= 1e-8) in fewer GMRES iterations."""

import numpy as np
import pytest
import torch

from conftest import golden
from paper_1602_05650_b200 import solver
from test_gpu_solver import aster_from

pytestmark = pytest.mark.gpu

CASES = {
    "step_aster.npz": lambda g: aster_from(g),
    "step_confined.npz": lambda g: aster_from(g, periphery=True, hinged=True),
}


def _probe(op, cols):
    n = op.layout.size
    e = torch.zeros(n, dtype=torch.float64, device=op.device)
    out = torch.empty((n, len(cols)), dtype=torch.float64, device=op.device)
    for k, j in enumerate(cols):
        e[j] = 1.0
        out[:, k] = op.rows_device(e, False)
        e[j] = 0.0
    return out


def _rel_max(a, b):
    return float((a - b).abs().max() / b.abs().max())


@pytest.mark.parametrize("name", sorted(CASES))
def test_particle_block_matrix_matches_probed_columns(cuda, name):
    g = golden(name)
    op, _ = solver.assemble_step_operator(CASES[name](g), float(g["dt"]))
    pend = op.layout.q1[-1].stop
    probed = _probe(op, range(pend))[:pend]
    assert _rel_max(op.particle_block_matrix(), probed) < 1e-12


@pytest.mark.parametrize("name", sorted(CASES))
def test_particle_rows_match_operator_rows(cuda, name):
    g = golden(name)
    op, _ = solver.assemble_step_operator(CASES[name](g), float(g["dt"]))
    lay = op.layout
    pend, fo = lay.q1[-1].stop, lay.fib_off
    y = torch.zeros(lay.size, dtype=torch.float64, device=op.device)
    y[fo:] = torch.as_tensor(np.random.default_rng(3).standard_normal(lay.size - fo),
                             device=op.device)
    full = op.rows_device(y, False)[:pend].clone()
    y[:fo] = 7.0            # surface entries of the input are ignored
    part = op.particle_rows_device(y)
    assert _rel_max(part, full) < 1e-13


@pytest.mark.parametrize("name", sorted(CASES))
def test_coupled_preconditioner_inverts_its_matrix(cuda, name):
    """z = P^-1 v with P = [[A_pp, A_pf], [A_f,Uomega, D_fibers]] (+ the
    periphery diagonal): P z reproduces v."""
    g = golden(name)
    op, _ = solver.assemble_step_operator(CASES[name](g), float(g["dt"]))
    lay = op.layout
    n, pend, fo = lay.size, lay.q1[-1].stop, lay.fib_off
    A = _probe(op, range(n))
    P = torch.zeros((n, n), dtype=torch.float64, device=op.device)
    P[:pend, :pend] = A[:pend, :pend]
    P[:pend, fo:] = A[:pend, fo:]
    P[fo:, :6] = A[fo:, :6]
    for m, sl in enumerate(lay.fiber_block):
        P[sl, sl] = op.fiber_blocks[m]
    prec = solver.Preconditioner(op, body_coupling=True)
    if lay.q0 is not None:
        idx = torch.arange(lay.q0.start, lay.q0.stop, device=op.device)
        P[idx, idx] = prec.diag[idx]
    v = torch.as_tensor(np.random.default_rng(5).standard_normal(n), device=op.device)
    z = prec.apply_device(v.clone())
    assert float((P @ z - v).norm() / v.norm()) < 1e-8


@pytest.mark.parametrize("name", sorted(CASES))
def test_body_coupled_steps_match_reference(cuda, name):
    g = golden(name)
    st = CASES[name](g)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    for s in range(int(g["nsteps"])):
        st, info = solver.backward_euler_step(st, float(g["dt"]), params, return_info=True,
                                              body_coupling=True)
        X = np.stack([f.X for f in st.fibers])
        ref = g[f"step{s}_X"]
        assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-8
        assert info["iterations"] < int(g[f"iters_{s}"])


def _two_asters():
    from paper_1602_05650_b200 import configs, system
    from paper_1602_05650_b200.fiber import ClampedToBody
    a = configs.aster(n_fibers=10, p=15, mesh_res=(4, 4), center=(-1.8, 0.0, 0.0), seed=1)
    b = configs.aster(n_fibers=8, p=15, mesh_res=(4, 4), center=(1.8, 0.2, 0.0), seed=2)
    for f in b.fibers:
        bc = f.bc_minus
        f.bc_minus = ClampedToBody(1, bc.attach_point, bc.tangent)
    return system.SystemState(a.fibers + b.fibers, a.particles + b.particles)


def test_two_particles_coupled_preconditioner(cuda):
    """Two asters: the Schur complement couples each particle to its own
    fibers; P z = v holds, and a step reproduces the block-Jacobi step's
    positions (<= 1e-9) in fewer iterations."""
    st = _two_asters()
    op, _ = solver.assemble_step_operator(st, 1e-3)
    lay = op.layout
    n, pend, fo = lay.size, lay.q1[-1].stop, lay.fib_off
    A = _probe(op, range(n))
    assert _rel_max(op.particle_block_matrix()[:lay.q1[0].stop, :lay.q1[0].stop],
                    A[:lay.q1[0].stop, :lay.q1[0].stop]) < 1e-12
    P = torch.zeros((n, n), dtype=torch.float64, device=op.device)
    B = op.particle_block_matrix()
    P[:pend, :pend] = B
    P[:pend, fo:] = A[:pend, fo:]
    for i in range(2):
        c = slice(lay.U[i].start, lay.U[i].start + 6)
        P[fo:, c] = A[fo:, c]
    for m, sl in enumerate(lay.fiber_block):
        P[sl, sl] = op.fiber_blocks[m]
    prec = solver.Preconditioner(op, body_coupling=True)
    v = torch.as_tensor(np.random.default_rng(9).standard_normal(n), device=op.device)
    z = prec.apply_device(v.clone())
    assert float((P @ z - v).norm() / v.norm()) < 1e-8
    params = solver.GmresParams(tolerance=1e-10)
    runs = {}
    for coupled in (False, True):
        s = _two_asters()
        s, info = solver.backward_euler_step(s, 1e-3, params, return_info=True,
                                             body_coupling=coupled)
        runs[coupled] = (np.concatenate([f.X for f in s.fibers]), info["iterations"])
    (x0, i0), (x1, i1) = runs[False], runs[True]
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x0) < 1e-9
    assert i1 < i0
