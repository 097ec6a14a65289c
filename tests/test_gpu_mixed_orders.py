"""Systems mixing Chebyshev orders (p = 15 and 23 interleaved), which the
reference supports fiber by fiber: operator, rhs, preconditioner and implicit
steps against the reference's own runs (golden step_mixed_*.npz).  Tolerances
as in test_gpu_solver.py."""

import numpy as np
import pytest

from conftest import golden
from oracle.ops import rel_l2
from paper_1602_05650_b200 import body, solver, system
from paper_1602_05650_b200.fiber import ClampedToBody, Fiber, PrescribedForceTorque

pytestmark = pytest.mark.gpu


def cloud(g):
    Xs = [g[f"init_X{k}"] for k in range(8)]
    return system.SystemState([Fiber(X, eps=5e-3, E=1e-2) for X in Xs],
                              force_models=[system.UniformBodyForce(1.0, (0.0, 0.0, -1.0))])


def aster(g):
    part = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4)))
    fibs = []
    o = 0
    for p in g["fiber_p"]:
        X = g["init_X"][o:o + p + 1]
        o += p + 1
        d = X[0] - X[-1]
        d = d / np.linalg.norm(d)
        fibs.append(Fiber(X, eps=1e-2, E=1.0, bc_minus=ClampedToBody(0, X[-1], d),
                          bc_plus=PrescribedForceTorque(1.0 * d)))
    return system.SystemState(fibs, [part])


CASES = {"step_mixed_cloud.npz": cloud, "step_mixed_aster.npz": aster}


@pytest.mark.parametrize("name", sorted(CASES))
def test_mixed_order_operator_and_steps(cuda, name):
    g = golden(name)
    st = CASES[name](g)
    op, rhs = solver.assemble_step_operator(st, float(g["dt"]))
    assert op.layout.size == int(g["layout_size"])
    assert len(op.batches) == 2
    assert rel_l2(op.apply(g["apply_u"]), g["apply_Au"]) < 1e-10
    assert rel_l2(rhs.cpu().numpy(), g["rhs"]) < 1e-10
    assert rel_l2(op.fiber_blocks[0].cpu().numpy(), g["block0"]) < 1e-11
    assert rel_l2(solver.Preconditioner(op).apply(g["prec_v"]), g["prec_Mv"]) < 1e-7
    params = solver.GmresParams(tolerance=float(g["tol"]))
    for s in range(int(g["nsteps"])):
        st, info = solver.backward_euler_step(st, float(g["dt"]), params, return_info=True)
        X = np.concatenate([f.X for f in st.fibers])
        ref = g[f"step{s}_X"]
        assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-8
        # tension of the p = 23 fibers is determined only to ~1e-4 by the
        # conditioning (D_s^4 ~ 1e10): under this operator the reference's own
        # solution has a true preconditioned residual of 4e-5 (ours 3e-6),
        # both after GMRES reported 1e-10; positions agree to 1e-10
        assert rel_l2(np.concatenate([f.T for f in st.fibers]), g[f"step{s}_T"]) < 1e-3
        assert abs(info["iterations"] - int(g[f"iters_{s}"])) <= 1
