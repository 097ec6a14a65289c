"""The per-constituent operator API a reference user calls directly
(fiber.py:237-289, body.py:237-283, 522-527), evaluated on the device,
against the reference's own outputs (golden api_ops.npz from
tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden
from oracle.ops import rel_l2
from paper_1602_05650_b200 import body, fiber

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    return golden("api_ops.npz")


def test_fiber_operators(cuda, g):
    fib = fiber.Fiber(g["X"], eps=float(g["eps"]), E=float(g["E"]))
    mu = float(g["mu"])
    assert rel_l2(fiber.elastic_force_density(fib, g["Xc"], g["Tc"]), g["elastic"]) < 1e-10
    assert rel_l2(fiber.local_mobility_apply(fib, g["f"], mu), g["mobility"]) < 1e-14
    assert rel_l2(fiber.nonlocal_Kdelta_apply(fib, g["f"], mu), g["kdelta"]) < 1e-12


def test_surface_operators(cuda, g):
    mu = float(g["mu"])
    per = body.make_surface(body.sphere_shape(3.0), (6, 6))
    part = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4)))
    part.F_ext, part.L_ext = g["F"], g["L"]
    assert rel_l2(body.double_layer_offsurface(per, g["q"], g["tgt"], mu), g["dl_off"]) < 1e-13
    assert rel_l2(body.double_layer_onsurface(per, g["q"], mu), g["dl_on"]) < 1e-13
    assert rel_l2(body.double_layer_onsurface(part.mesh, g["qp"], mu), g["dl_on_p"]) < 1e-13
    assert rel_l2(body.completion_flow(part, g["tgt"] + 1.0, mu), g["completion"]) < 1e-14
    assert rel_l2(body.near_surface_eval(per, g["q"], g["near_t"], mu), g["near_eval"]) < 1e-11


def test_near_shell_is_enforced(cuda, g):
    from paper_1602_05650_b200 import kernels
    per = body.make_surface(body.sphere_shape(3.0), (6, 6))
    with pytest.raises(kernels.NearFieldError):
        body.double_layer_offsurface(per, g["q"], g["near_t"][None, :], float(g["mu"]))


def test_fiber_kdelta_matrix_method(cuda, g):
    fib = fiber.Fiber(g["X"], eps=float(g["eps"]), E=float(g["E"]))
    assert np.array_equal(fib.kdelta_matrix(float(g["mu"])), g["Kmat"])   # bitwise build


def test_surface_helpers(cuda, g):
    """second_kind_matrix (device assembly), interpolate_nodal, and the
    reference-named near_surface_weights (body.py:316-566)."""
    mu = float(g["mu"])
    per = body.make_surface(body.sphere_shape(3.0), (6, 6))
    A = body.second_kind_matrix(body.make_surface(body.sphere_shape(0.5), (2, 2)), mu,
                                interior=False)
    assert np.abs(A - g["skm"]).max() <= 1e-13 * np.abs(g["skm"]).max()
    A = body.second_kind_matrix(body.make_surface(body.sphere_shape(3.0), (2, 2)), mu,
                                interior=True, nullspace_scale=0.5)
    assert np.abs(A - g["skm_per"]).max() <= 1e-13 * np.abs(g["skm_per"]).max()
    got = body.interpolate_nodal(per, g["q"], np.array([0.3, 1.7, 2.9]), np.array([0.1, 3.0, 6.1]))
    assert np.array_equal(got, g["interp"])
    W = body.near_surface_weights(per, g["near_t"], mu, interior_jump=True)
    assert np.abs(W - g["near_W"]).max() <= 1e-12 * np.abs(g["near_W"]).max()


def test_fiber_near_field_api(cuda, g):
    """near_fiber_weights / near_fiber_eval (device-built map) and
    resample_to_fine against the reference (fiber.py:444-587)."""
    fib = fiber.Fiber(g["X"], eps=float(g["eps"]), E=float(g["E"]))
    mu = float(g["mu"])
    W = fiber.near_fiber_weights(fib, g["fnear_t"], mu, include_doublet=True)
    assert np.abs(W - g["fnear_W"]).max() <= 1e-11 * np.abs(g["fnear_W"]).max()
    assert rel_l2(fiber.near_fiber_eval(fib, g["f"], g["fnear_t"], mu), g["fnear_eval"]) < 1e-11
    assert np.array_equal(fiber.resample_to_fine(g["f"][:, 0], np.linspace(-1, 1, 7)),
                          g["resampled"])


def test_kernel_helpers(cuda, g):
    """rotlet_sum (device) and the single-pair *_apply helpers (kernels.py:22-174).
    The host boundary residuals (fiber.py:375-441) stay in the reference; the
    device rows that replace them are pinned through BlockOperator.apply
    (test_gpu_solver.py, test_gpu_baseline_steps.py)."""
    from paper_1602_05650_b200 import kernels
    mu = float(g["mu"])
    rot, bad = kernels.rotlet_sum(g["tgt"], g["rot_src"], g["rot_L"], 0.2)
    assert bad == 0 and rel_l2(rot, g["rot"]) < 1e-14
    f, t = g["f"], g["tgt"]
    a = np.concatenate([kernels.stokeslet_apply(t[0], f[0], mu),
                        kernels.stresslet_apply(t[0], f[1], f[2], mu),
                        kernels.rotlet_apply(t[1], f[3], mu), kernels.doublet_apply(t[2], f[4], mu)])
    assert np.array_equal(a, g["apply1"])

