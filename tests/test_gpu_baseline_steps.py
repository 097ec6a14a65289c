"""Implicit steps at the BASELINE orders and step counts against the
reference's own trajectories (tests/golden/make_golden_baseline.py, made by
running slenderflow): C1 as 10 steps (p = 31, near-field maps rebuilt every
step), a 256-fiber C2 aster for 10 steps, the full 1,024-fiber C2 aster for
2 steps, a p = 63 C3 cloud for 20 steps and a C4 confined aster in the
40,960-node periphery for 5 steps.

Tolerances (north_star): operator A u and rhs <= 1e-10 relative L2;
preconditioner M v <= 1e-7 (equilibrated block LU, cond ~1e8 at p = 31;
at p = 63 20x the reference's own first-step M v sensitivity);
positions <= 1e-8 relative after every step; GMRES iteration counts within
one of the reference's.  Where the reference's OWN trajectory is not fixed
to that level by FP64, the bound is 20x its measured rounding sensitivity
(tests/golden/tension_sensitivity.json: the reference re-run from
centrelines changed by 1e-15 relative).  That is the case for the tensions
and surface densities at every step (the inextensibility rows are D_s^4 sums
of size ~1e12 cancelling to O(1): T moves 2e-4-8e-4, q1 1e-7-1e-5) and
for the positions of the C1 near-pair cloud after its first step (1e-7 at
step 1 growing to 5e-6 by step 6: the near-field quadrature's adaptive panel
splits and nearest-point searches are discrete decisions that rounding can
flip), and for everything at p = 63: there the reference's own positions
move by 8e-7 after the first step and its tensions by 20-100 %."""

import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle.ops import rel_l2
from paper_1602_05650_b200 import body, solver, system
from paper_1602_05650_b200.fiber import ClampedToBody, Fiber, PrescribedForceTorque

pytestmark = pytest.mark.gpu

CASES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "bstep_*.npz")))
SENS = json.load(open(os.path.join(GOLDEN, "tension_sensitivity.json")))


# full-size trajectory fixtures use the sensitivity measured on their
# reduced-size analogue (same physics; re-running the reference twice more
# at full size would take hours): the 256-fiber aster for the 10-step C2,
# the 128-fiber confined aster for C4
SENS_PROXY = {"bstep_c2_10": "bstep_aster256", "bstep_c4": "bstep_confined"}


def sens_tol(name, step, key, base):
    """max(base, 20x the reference's own change of `key` after `step` under
    a 1e-15 relative input perturbation)."""
    rec = SENS.get(SENS_PROXY.get(name[:-4], name[:-4]))
    if rec is None:
        return base
    steps = rec.get("steps", [])
    if step < len(steps) and key in steps[step]:
        return max(base, 20.0 * steps[step][key])
    vals = [s[key] for s in steps if key in s] or ([rec["d" + key]] if "d" + key in rec else [])
    return max(base, 20.0 * max(vals)) if vals else base


def _light(g):
    return "light" in g


def op_tol(name, key, base):
    """max(base, 20x the change of the reference's first-step A u / rhs / M v
    under the 1e-15 input perturbation).  At p = 63 the equilibrated fiber
    blocks are so ill-conditioned that the reference's own M v moves at the
    1e-6-1e-5 level."""
    rec = SENS.get(name[:-4], {}).get("operator", {})
    return max(base, 20.0 * rec[key]) if key in rec else base


def state_from(g):
    """The fixture's initial state built with this package's constructors
    from the same arrays the reference was given."""
    kind = str(g["spec_kind"])
    eps, E = float(g["spec_eps"]), float(g["spec_E"])
    if kind == "cloud":
        fibs = [Fiber(X, eps=eps, E=E) for X in g["init_X"]]
        return system.SystemState(fibs, force_models=[system.UniformBodyForce(
            float(g["spec_f0"]), tuple(g["spec_direction"]))])
    center = tuple(float(c) for c in g["spec_center"])
    part = body.RigidParticle(body.make_surface(body.sphere_shape(float(g["spec_radius"])),
                                                tuple(int(r) for r in g["spec_mesh_res"]),
                                                center=center))
    motor = float(g["spec_motor"])
    fibs = [Fiber(X, eps=eps, E=E, bc_minus=ClampedToBody(0, x0, d),
                  bc_plus=PrescribedForceTorque(motor * d))
            for X, x0, d in zip(g["init_X"], g["att_x"], g["att_d"])]
    per = None
    if float(g["spec_per_radius"]) > 0:
        per = body.Periphery(body.make_surface(body.sphere_shape(float(g["spec_per_radius"])),
                                               tuple(int(r) for r in g["spec_per_res"])))
    return system.SystemState(fibs, [part], per)


def test_fixtures_present():
    assert {"bstep_c1.npz", "bstep_aster256.npz", "bstep_confined.npz"} <= set(CASES)


@pytest.mark.parametrize("name", CASES)
def test_operator_rhs_preconditioner_at_baseline_orders(cuda, name):
    g = golden(name)
    if _light(g):
        pytest.skip("trajectory-only fixture (operator records live in its reduced analogue)")
    st = state_from(g)
    op, rhs = solver.assemble_step_operator(st, float(g["dt"]))
    n = op.layout.size
    assert n == int(g["layout_size"])
    u = np.random.default_rng(int(g["seed_u"])).standard_normal(n)
    v = np.random.default_rng(int(g["seed_v"])).standard_normal(n)
    assert rel_l2(op.apply(u), g["apply_Au"]) < op_tol(name, "Au", 1e-10)
    assert rel_l2(rhs.cpu().numpy(), g["rhs"]) < op_tol(name, "rhs", 1e-10)
    assert len(op.cache.near_fiber) == int(g["n_near_fiber"])
    assert len(op.cache.near_surface) == int(g["n_near_surface"])
    assert rel_l2(solver.Preconditioner(op).apply(v), g["prec_Mv"]) < op_tol(name, "Mv", 1e-7)


@pytest.mark.parametrize("name", CASES)
def test_trajectory_matches_reference_every_step(cuda, name):
    g = golden(name)
    st = state_from(g)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    for s in range(int(g["nsteps"])):
        st, info = solver.backward_euler_step(st, float(g["dt"]), params, return_info=True)
        X = np.stack([f.X for f in st.fibers])
        ref = g[f"step{s}_X"]
        err = np.linalg.norm(X - ref) / np.linalg.norm(ref)
        assert err <= sens_tol(name, s, "X", 1e-8), (s, err)
        assert abs(info["iterations"] - int(g[f"iters_{s}"])) <= 1, (s, info["iterations"])
        assert abs(st.time - float(g[f"time_{s}"])) <= 1e-15
        if f"step{s}_T" in g:
            T = np.stack([f.T for f in st.fibers])
            assert rel_l2(T, g[f"step{s}_T"]) < sens_tol(name, s, "T", 1e-6), s
        if st.particles:
            U = np.stack([p.U for p in st.particles])
            assert rel_l2(U, g[f"step{s}_U"]) < sens_tol(name, s, "U", 1e-6), s
            q1 = np.stack([p.q for p in st.particles])
            assert rel_l2(q1, g[f"step{s}_q1"]) < sens_tol(name, s, "q1", 1e-6), s
    last = int(g["nsteps"]) - 1
    if f"step{last}_q0" in g:
        assert rel_l2(np.asarray(st.periphery.q), g[f"step{last}_q0"]) < \
            sens_tol(name, last, "q0", 1e-6)
