"""The drop-in, exercised on the REAL reference package.

`slenderflow` itself (installed unmodified into baseline/_ref by build(), the
reference arm's sanctioned install) is imported and its kernel seam rebound
to this package's C-ABI entry points: every caller in slenderflow resolves
`kernels.<fn>` at call time (system.py:99,198,215,665,680; fiber.py:217,
278,284; body.py:246,261,431; solver.py:411,416), so after the rebinding
slenderflow's own complementary_velocities, BlockOperator, Preconditioner
and backward_euler_step run their pair sums and K_delta builds on the B200.
The summation backend is passed as this package's DeviceSummation
(system.py:93-105).  Results are compared with golden vectors made by the
unmodified reference (tests/golden/make_golden.py): operator outputs
<= 1e-10 relative, positions <= 1e-8.

Skipped only when baseline/_ref has not been staged (build() does it
whenever /root/reference is present)."""

import importlib
import os
import sys

import numpy as np
import pytest

from conftest import golden
from oracle.ops import rel_l2

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SEAM = ("stokeslet_sum", "doublet_sum", "stresslet_sum", "stresslet_sum_subtracted",
        "stresslet_rowsum", "kdelta_matrix")


@pytest.fixture(scope="module")
def sf():
    if not os.path.isdir(os.path.join(REF, "slenderflow")):
        pytest.skip("reference not staged in baseline/_ref (run __graft_entry__.build())")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_dropin")
    sys.path.insert(0, REF)
    try:
        mods = {m: importlib.import_module(f"slenderflow.{m}")
                for m in ("kernels", "system", "solver", "fiber", "body")}
    finally:
        sys.path.remove(REF)
    assert mods["kernels"].__file__.startswith(REF)
    return mods


@pytest.fixture
def rebound(sf, monkeypatch, cuda):
    """slenderflow.kernels.<fn> -> paper_1602_05650_b200.kernels.<fn> (numpy in,
    numpy out, host-buffer C ABI), for the duration of one test."""
    from paper_1602_05650_b200 import kernels as ours
    calls = {k: 0 for k in SEAM}
    for name in SEAM:
        fn = getattr(ours, name)

        def wrapped(*a, _fn=fn, _name=name):
            calls[_name] += 1
            return _fn(*a)
        monkeypatch.setattr(sf["kernels"], name, wrapped)
    return calls


def test_reference_complementary_velocities_on_the_device(sf, rebound):
    """slenderflow.system.complementary_velocities on C1 (64 fibers, p = 31,
    18 near pairs) with its kernel seam on the B200 and the backend
    DeviceSummation: equals the unmodified reference's u_nl."""
    from paper_1602_05650_b200.system import DeviceSummation
    g = golden("c1_near.npz")
    F = sf["fiber"]
    fibs = [F.Fiber(X, eps=float(g["eps"]), E=float(g["E"])) for X in g["X"]]
    st = sf["system"].SystemState(fibs, mu=float(g["mu"]))
    res = sf["system"].complementary_velocities(st, fiber_forces=list(g["forces"]),
                                                backend=DeviceSummation())
    u = np.concatenate(res.fibers)
    assert rel_l2(u, g["u_nl"]) <= 1e-10
    assert rebound["doublet_sum"] >= 1          # the doublet pass went through the seam


def test_reference_step_on_the_device(sf, rebound):
    """slenderflow.solver.backward_euler_step on the golden aster (12 clamped
    fibers on a particle, p = 15) for its 2 steps, with the seam rebound and
    backend=DeviceSummation(): positions <= 1e-8, iteration counts equal."""
    from paper_1602_05650_b200.system import DeviceSummation
    g = golden("step_aster.npz")
    F, B, S = sf["fiber"], sf["body"], sf["system"]
    part = B.RigidParticle(B.make_surface(B.sphere_shape(0.5), (4, 4)))
    fibs = []
    for X in g["init_X"]:
        d = X[0] - X[-1]
        d = d / np.linalg.norm(d)
        fibs.append(F.Fiber(X, eps=1e-2, E=1.0, bc_minus=F.ClampedToBody(0, X[-1], d),
                            bc_plus=F.PrescribedForceTorque(1.0 * d)))
    st = S.SystemState(fibs, [part])
    solver = sf["solver"]
    iters = []
    orig = solver.gmres_solve

    def counting(*a, **k):
        out = orig(*a, **k)
        iters.append(out[1])
        return out
    solver.gmres_solve = counting
    try:
        params = solver.GmresParams(tolerance=float(g["tol"]))
        for s in range(int(g["nsteps"])):
            solver.backward_euler_step(st, float(g["dt"]), params, backend=DeviceSummation())
            X = np.stack([f.X for f in st.fibers])
            ref = g[f"step{s}_X"]
            assert np.linalg.norm(X - ref) / np.linalg.norm(ref) <= 1e-8, s
            assert iters[-1] == int(g[f"iters_{s}"]), (s, iters[-1])
    finally:
        solver.gmres_solve = orig
    assert rebound["kdelta_matrix"] >= 1 and rebound["stresslet_sum_subtracted"] >= 1
