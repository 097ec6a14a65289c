"""Implicit steps with polymerization kinetics and contact models
(solver.py:574-588, fiber.py:297-356, system.py:334-388): the device solve
with the Ldot reparametrization in its rows, then the reference's per-fiber
transitions with the same RNG streams, against the reference's own runs
(golden step_pushing.npz / step_pulling.npz)."""

import numpy as np
import pytest

from conftest import golden
from oracle.ops import rel_l2
from paper_1602_05650_b200 import body, fiber, solver, system

pytestmark = pytest.mark.gpu

KIN = dict(v_grow=0.5, v_shrink=0.8, f_cat=150.0, f_res=250.0, stall_force=4.4, min_length=0.5)


def build(g, pushing):
    pnc = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4)))
    fibs = []
    for k, (X, d) in enumerate(zip(g["init_X"], g["init_d"])):
        fibs.append(fiber.Fiber(X, eps=1e-2, E=1.0, growth_state=fiber.GROWING, Ldot=KIN["v_grow"],
                                rng=np.random.default_rng(100 + k),
                                kinetics=fiber.GrowthKinetics(**KIN),
                                bc_minus=fiber.ClampedToBody(0, X[-1], d)))
    per = body.Periphery(body.make_surface(body.sphere_shape(1.8), (6, 6)))
    models = ([system.CorticalPushing(stiffness=5.0, contact_distance=0.2, tau_cat=0.5)] if pushing
              else [system.CytoplasmicPulling(motor_force=0.91, motor_density=0.5)])
    return system.SystemState(fibs, [pnc], per, force_models=models)


@pytest.mark.parametrize("name,pushing", [("step_pushing.npz", True), ("step_pulling.npz", False)])
def test_kinetics_steps_match_reference(cuda, name, pushing):
    g = golden(name)
    st = build(g, pushing)
    params = solver.GmresParams(tolerance=1e-10)
    for s in range(int(g["nsteps"])):
        st = solver.backward_euler_step(st, float(g["dt"]), params)
        assert [f.growth_state for f in st.fibers] == list(g[f"step{s}_state"])
        assert [f.bc_plus.kind for f in st.fibers] == list(g[f"step{s}_bcplus"])
        assert np.allclose([f.tau_cat for f in st.fibers], g[f"step{s}_tau"])
        Ld = np.array([f.Ldot for f in st.fibers])
        assert np.abs(Ld - g[f"step{s}_Ldot"]).max() <= 1e-8
        X = np.stack([f.X for f in st.fibers])
        ref = g[f"step{s}_X"]
        assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-8
        assert rel_l2(np.stack([f.T for f in st.fibers]), g[f"step{s}_T"]) < 1e-6
