"""The reference's analytic and structural test identities, re-asserted on the
device path (test_system.py, test_fiber.py, test_body.py of the reference;
tolerances as there unless noted)."""


import numpy as np
import pytest

from oracle import ops
from paper_1602_05650_b200 import body, kernels, system
from paper_1602_05650_b200.fiber import straight_fiber
from paper_1602_05650_b200.operator import FiberHIOperator

pytestmark = pytest.mark.gpu


def zfiber(base, length=2.0, p=12, **kw):
    return straight_fiber(p, base, (0.0, 0.0, 1.0), length, **kw)


def test_mirrored_pair_is_symmetric(cuda):
    # test_system.py:130-139
    fa = zfiber((1.0, 0.2, -1.0))
    fb = zfiber((-1.0, 0.2, -1.0))
    f = np.tile([0.0, 0.3, 1.0], (13, 1))
    res = system.complementary_velocities(system.SystemState([fa, fb]), fiber_forces=[f, f])
    mirror = np.array([-1.0, 1.0, 1.0])
    scale = np.abs(res.fibers[0]).max()
    assert scale > 0
    assert np.abs(res.fibers[1] - mirror * res.fibers[0]).max() <= 1e-12 * scale


def test_far_pair_matches_slender_body_quadrature(cuda):
    # test_system.py:141-150: equals the fiber's induced flow with the doublet
    fa = zfiber((0, 0, -1.0))
    fb = zfiber((5.0, 0, -1.0))
    f = np.random.default_rng(3).standard_normal((13, 3))
    res = system.complementary_velocities(system.SystemState([fa, fb]),
                                          fiber_forces=[f, np.zeros((13, 3))])
    w = fa.node_weights()
    coeff = (fa.eps * fa.L) ** 2 / 2.0
    st, _ = kernels.stokeslet_sum(fb.X, None, fa.X, None, w[:, None] * f, 1 / (8 * np.pi))
    db, _ = kernels.doublet_sum(fb.X, None, fa.X, None, w[:, None] * f, coeff / (8 * np.pi))
    assert np.abs(res.fibers[1] - (st + db)).max() < 1e-14
    assert np.all(res.fibers[0] == 0.0)


def test_stokeslet_reciprocity(cuda):
    # test_system.py:152-162
    fa = straight_fiber(12, (0, 0, -1.0), (0, 0, 1.0), 2.0)
    fb = straight_fiber(12, (3.0, 1.0, 0.2), (0.6, 0.8, 0.0), 2.0)
    rng = np.random.default_rng(7)
    f1, f2 = rng.standard_normal((13, 3)), rng.standard_normal((13, 3))
    res = system.complementary_velocities(system.SystemState([fa, fb]), fiber_forces=[f1, f2],
                                          include_doublet=False)
    s_ab = float(np.sum(fb.node_weights()[:, None] * f2 * res.fibers[1]))
    s_ba = float(np.sum(fa.node_weights()[:, None] * f1 * res.fibers[0]))
    assert abs(s_ab - s_ba) <= 1e-10 * max(abs(s_ab), 1.0)


def test_kdelta_annihilates_constants_on_straight_fiber(cuda):
    # test_fiber.py:138-143: K_delta f = 0 for constant f on a straight fiber;
    # the device self term then equals the local mobility alone
    f0 = straight_fiber(24, (0, 0, 0), (1, 0, 0), 2.0)
    op = FiberHIOperator(f0.X[None], f0.eps)
    for force in ([1.0, 0, 0], [0, 1.0, 0], [0.3, -0.2, 0.9]):
        F = np.tile(force, (1, 25, 1))
        _, u_self = op.apply(F)
        mob = ops.local_mobility_apply(f0.tangents, f0.eps, F[0], 1.0)
        assert np.abs(u_self.cpu().numpy() - mob).max() < 1e-12


def test_kdelta_linear_force_oracle(cuda):
    # test_fiber.py:145-155 (explicit delta = 0.05)
    L = 2.0
    fib = straight_fiber(32, (0, 0, 0), (1, 0, 0), L)
    op = FiberHIOperator(fib.X[None], fib.eps, delta=0.05)
    force = np.stack([np.zeros_like(fib.s), fib.s, np.zeros_like(fib.s)], axis=1)
    _, u_self = op.apply(force[None])
    mob = ops.local_mobility_apply(fib.tangents, fib.eps, force, 1.0)
    v = (u_self.cpu().numpy() - mob) * (8.0 * np.pi)
    d = 0.05
    expect = np.sqrt((L - fib.s) ** 2 + d ** 2) - np.sqrt(fib.s ** 2 + d ** 2)
    mid = fib.n_nodes // 2
    assert v[mid, 1] == pytest.approx(expect[mid], abs=2e-2 * L)


def test_double_layer_interior_constant_identity(cuda):
    # test_body.py:98-106: interior value of a constant density is q/mu, exterior 0
    mesh = body.make_surface(body.sphere_shape(1.0), (8, 8))
    q = np.tile([0.4, -0.7, 0.2], (mesh.n_nodes, 1))
    mu = 2.0
    qw = q * mesh.weights[:, None]
    pref = -3.0 / (4.0 * np.pi * mu)
    inside, _ = kernels.stresslet_sum(np.array([[0.1, -0.2, 0.3]]), None, mesh.nodes, None,
                                      mesh.normals, qw, pref)
    assert np.allclose(inside[0], np.array([0.4, -0.7, 0.2]) / mu, atol=1e-8)
    outside, _ = kernels.stresslet_sum(np.array([[4.0, 1.0, -2.0]]), None, mesh.nodes, None,
                                       mesh.normals, qw, pref)
    assert np.abs(outside).max() < 1e-8


def test_near_surface_routing_and_interior_jump(cuda):
    # test_system.py:209-219: a fiber tip next to the periphery sees q/mu
    per = body.Periphery(body.make_surface(body.sphere_shape(6.0), (12, 12)))
    fib = zfiber((0, 0, 2.2), length=3.3)
    st = system.SystemState([fib], periphery=per)
    q = np.tile([0.1, -0.2, 0.3], (per.mesh.n_nodes, 1))
    cache = system.InteractionCache(st)
    assert len(cache.near_surface) > 0
    res = system.complementary_velocities(st, periphery_density=q, fiber_forces=[np.zeros((13, 3))],
                                          cache=cache)
    assert np.abs(res.fibers[0][0] - q[0] / st.mu).max() < 1e-7
