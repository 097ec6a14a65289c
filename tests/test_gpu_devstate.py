"""The step state lives on the device between implicit steps
(devstate.DeviceState): reading a host attribute brings the state back,
writing one hands it back to the host, and neither changes the trajectory."""

import copy

import numpy as np
import pytest

from conftest import golden
from paper_1602_05650_b200 import devstate, solver
from test_gpu_solver import CASES

pytestmark = pytest.mark.gpu


def _X(st):
    return np.stack([f.X for f in st.fibers])


def test_device_state_is_used_between_steps_and_read_lazily(cuda):
    g = golden("step_aster.npz")
    st = CASES["step_aster.npz"](g)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    dt = float(g["dt"])
    solver.backward_euler_step(st, dt, params)
    mirror = devstate.mirror_of(st)
    assert mirror is not None and mirror.stale          # host copies not refreshed yet
    # nothing host-side was touched: the second step reuses the device state
    solver.backward_euler_step(st, dt, params)
    assert devstate.mirror_of(st) is mirror
    X = _X(st)                                           # first read pulls everything
    assert not mirror.stale
    assert np.linalg.norm(X - g["step1_X"]) / np.linalg.norm(g["step1_X"]) < 1e-8
    p = st.particles[0]
    ref_U = g["step1_U"][0]
    assert np.linalg.norm(p.U - ref_U) <= 1e-6 * np.linalg.norm(ref_U)
    assert p.mesh.nodes.shape == (p.mesh.n_nodes, 3)
    # the particle translated by dt U in both steps (RigidParticle.translate)
    assert np.linalg.norm(p.center) > 0


def test_host_writes_hand_the_state_back(cuda):
    """Writing fib.X between steps releases the device state; the next step
    starts from the host values, exactly like a fresh state built from them."""
    g = golden("step_cloud.npz")
    st = CASES["step_cloud.npz"](g)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    dt = float(g["dt"])
    solver.backward_euler_step(st, dt, params)
    shifted = _X(st) + np.array([1e-3, 0.0, 0.0])
    fresh = copy.deepcopy(st)
    for f, X in zip(st.fibers, shifted):
        f.X = X                                          # host write: mirror released
    assert devstate.mirror_of(st) is None
    for f, X in zip(fresh.fibers, shifted):
        f.X = X
    solver.backward_euler_step(st, dt, params)
    solver.backward_euler_step(fresh, dt, params)
    assert np.array_equal(_X(st), _X(fresh))
    assert np.array_equal(np.stack([f.T for f in st.fibers]),
                          np.stack([f.T for f in fresh.fibers]))


def test_mirror_matches_a_host_round_trip_bitwise(cuda):
    """Stepping with the device state kept between steps equals stepping
    with the state forced back to the host after every step (release),
    bit for bit."""
    g = golden("step_confined.npz")
    st_a = CASES["step_confined.npz"](g)
    st_b = copy.deepcopy(st_a)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    dt = float(g["dt"])
    for _ in range(2):
        solver.backward_euler_step(st_a, dt, params)
        solver.backward_euler_step(st_b, dt, params)
        devstate.mirror_of(st_b).release()               # host round trip every step
    assert np.array_equal(_X(st_a), _X(st_b))
    assert np.array_equal(np.asarray(st_a.periphery.q), np.asarray(st_b.periphery.q))
