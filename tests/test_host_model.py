"""Host-side setup code (meshes, fibers) and the oracle's host near-field maps
(oracle/nearfield.py, the checker of the device construction) against the
reference's own outputs (golden fixtures)."""

import numpy as np
import pytest

from conftest import golden
from oracle import nearfield
from paper_1602_05650_b200 import body
from paper_1602_05650_b200.fiber import Fiber, straight_fiber


def test_surface_meshes_bitwise():
    g = golden("surfaces.npz")
    per = body.make_surface(body.sphere_shape(6.0), (8, 8))
    part = body.make_surface(body.sphere_shape(1.0), (6, 6))
    for m, k in ((per, "per"), (part, "part")):
        assert np.array_equal(m.nodes, g[f"{k}_nodes"])
        assert np.array_equal(m.normals, g[f"{k}_normals"])
        assert np.array_equal(m.weights, g[f"{k}_weights"])


def test_fiber_geometry_matches_reference():
    g = golden("c1_near.npz")
    for m in (0, 17, 63):
        fib = Fiber(g["X"][m], eps=float(g["eps"]), E=1.0)
        assert np.array_equal(fib.s_alpha, g["s_alpha"][m])
        assert np.abs(fib.s - g["s"][m]).max() < 1e-15
        assert np.abs(fib.tangents - g["tangents"][m]).max() < 1e-15
        assert np.abs(fib.node_weights() - g["weights"][m]).max() < 1e-16
        assert fib.delta == g["delta"][m]


def test_straight_fiber_layout():
    f = straight_fiber(31, (0.1, 0.2, 0.3), (1, 2, 3), 1.0)
    assert np.allclose(f.X[-1], (0.1, 0.2, 0.3)) and f.end_index(False) == 31
    assert abs(f.L - 1.0) < 1e-12


def test_near_fiber_maps_match_reference():
    g = golden("c1_near.npz")
    fibers = [Fiber(X, eps=float(g["eps"]), E=1.0) for X in g["X"]]
    targets = g["X"].reshape(-1, 3)
    groups = np.repeat(np.arange(len(fibers)), g["X"].shape[1])
    near = nearfield.find_fiber_pairs(fibers, targets, groups, float(g["mu"]), True)
    assert [(t, l) for t, l, _ in near] == list(zip(g["near_t"].tolist(), g["near_l"].tolist()))
    for (_, _, W), Wref in zip(near, g["near_W"]):
        assert np.abs(W - Wref).max() <= 1e-12 * np.abs(Wref).max()


def test_near_surface_maps_match_reference():
    g = golden("near_surface.npz")
    part = body.make_surface(body.sphere_shape(0.5), (4, 4))
    per = body.make_surface(body.sphere_shape(3.0), (6, 6))
    for t, Wref in zip(g["tp"], g["Wp"]):
        W = nearfield.near_surface_weights(part, t, 1.0, interior_jump=False) \
            - nearfield.plain_surface_weights(part, t, 1.0)
        assert np.abs(W - Wref).max() <= 1e-12 * np.abs(Wref).max()
    for t, Wref, ns in zip(g["tq"], g["Wq"], g["nsp"]):
        th, ph, x0, d = nearfield.nearest_surface_point(per, t)
        assert abs(th - ns[0]) < 1e-12 and abs(d - ns[5]) < 1e-12
        W = nearfield.near_surface_weights(per, t, 1.0, interior_jump=True) \
            - nearfield.plain_surface_weights(per, t, 1.0)
        assert np.abs(W - Wref).max() <= 1e-12 * np.abs(Wref).max()


def test_tree_topology_partitions_the_points():
    """tree.build_topology: every node owns a contiguous permuted range that
    its children tile in octant order; leaves hold <= leaf_size points."""
    from paper_1602_05650_b200 import tree
    rng = np.random.default_rng(0)
    pts = np.vstack([rng.standard_normal((500, 3)), rng.standard_normal((300, 3)) + 8.0])
    perm, nb, ne, first, nch = tree.build_topology(pts, 16)
    assert sorted(perm.tolist()) == list(range(pts.shape[0]))
    assert nb[0] == 0 and ne[0] == pts.shape[0]
    for k in range(nb.size):
        if nch[k] == 0:
            assert ne[k] - nb[k] <= 16
            assert list(perm[nb[k]:ne[k]]) == sorted(perm[nb[k]:ne[k]])   # reference idx order
        else:
            kids = range(first[k], first[k] + nch[k])
            assert nb[first[k]] == nb[k] and ne[first[k] + nch[k] - 1] == ne[k]
            assert all(ne[a] == nb[a + 1] for a in list(kids)[:-1])


def test_profile_shape_meshes_match_reference():
    """s1/s2/s3 profile meshes (body.py:37-72) bitwise equal to the reference's."""
    g = golden("shapes.npz")
    for k in ("s1", "s2", "s3"):
        m = body.make_surface(body.named_shape(k, 2.0), (6, 8), center=(0.1, -0.2, 0.3))
        assert np.array_equal(m.nodes, g[f"{k}_nodes"])
        assert np.array_equal(m.normals, g[f"{k}_normals"])
        assert np.array_equal(m.weights, g[f"{k}_weights"])
    per = body.make_surface(body.s1_shape(2.0), (6, 8))
    for t, ns in zip(g["near_t"], g["near_ns"]):
        th, ph, _, d = nearfield.nearest_surface_point(per, t)
        assert abs(th - ns[0]) < 1e-12 and abs(d - ns[2]) < 1e-12


def test_spectral_api_matches_reference():
    """ChebyshevGrid, arclength_map and the cheb_* helpers bitwise equal to
    the reference's (spectral.py:24-154)."""
    from paper_1602_05650_b200 import spectral as S
    g = golden("spectral.npz")
    grid = S.ChebyshevGrid(31)
    for k in ("nodes", "weights", "D"):
        assert np.array_equal(getattr(grid, k), g[k])
    s, sa, L = S.arclength_map(g["X"], grid)
    assert np.array_equal(s, g["s"]) and np.array_equal(sa, g["s_alpha"]) and L == float(g["L"])
    assert np.array_equal(S.cheb_diff(g["v"], grid), g["dv"])
    assert S.cheb_integrate(g["v"], grid) == float(g["iv"])
    assert np.array_equal(S.cheb_transform(g["v"]), g["cv"])
    assert np.array_equal([S.cheb_interp(g["v"], a) for a in (-1.0, -0.37, 0.3, 1.0)], g["interp"])
    with pytest.raises(S.InvalidOrderError):
        S.ChebyshevGrid(3)


def test_gmres_params_validation():
    from paper_1602_05650_b200 import solver, system
    for kw in (dict(tolerance=0.0), dict(tolerance=1.0), dict(restart=0), dict(max_iterations=0)):
        with pytest.raises(system.ConfigurationError):
            solver.GmresParams(**kw)


def test_fiber_dense_operators_match_reference():
    """Fiber.Ds..Ds4, elastic_operators, mobility_matrix and the grid object
    (fiber.py:133-222) equal the reference's bitwise."""
    g = golden("api_ops.npz")
    fib = Fiber(g["X"], eps=float(g["eps"]), E=float(g["E"]))
    assert np.array_equal(fib.Ds4, g["Ds4"])
    FX, FT = fib.elastic_operators()
    assert np.array_equal(FX, g["FX"]) and np.array_equal(FT, g["FT"])
    assert np.array_equal(fib.mobility_matrix(float(g["mu"])), g["Mmat"])
    assert fib.grid.p == fib.p and fib.grid.D.shape == (fib.n_nodes, fib.n_nodes)


def test_warm_start_vector_round_trips_through_the_layout():
    """solver.warm_start_vector packs the state in StepLayout order
    (solver.py:67-110): unpack returns the state's own arrays."""
    from paper_1602_05650_b200 import configs, solver
    st = configs.aster(n_fibers=6, p=15, mesh_res=(4, 4))
    rng = np.random.default_rng(0)
    part = st.particles[0]
    part.U, part.omega = rng.standard_normal(3), rng.standard_normal(3)
    part.q = rng.standard_normal(part.q.shape)
    for f in st.fibers:
        f.T = rng.standard_normal(f.T.shape)
    lay = solver.StepLayout(st)
    parts = lay.unpack(solver.warm_start_vector(st, lay))
    assert np.array_equal(parts.U[0], part.U) and np.array_equal(parts.omega[0], part.omega)
    assert np.array_equal(parts.q1[0], part.q)
    for m, f in enumerate(st.fibers):
        assert np.array_equal(parts.X[m], f.X) and np.array_equal(parts.T[m], f.T)


def test_icosphere_mesh():
    """make_icosphere (BASELINE config 4's literal 40,962-vertex mesh): vertex
    count 10 * 4^k + 2, nodes on the sphere, radial unit normals, weights
    summing to the sphere's area, accepted as a periphery."""
    import math
    m = body.make_icosphere(2.0, 6)
    assert m.n_nodes == 40962 and m.triangles.shape == (20 * 4 ** 6, 3)
    assert np.allclose(np.linalg.norm(m.nodes, axis=1), 2.0, atol=1e-14)
    assert np.allclose(m.normals, m.nodes / 2.0, atol=1e-15)
    assert abs(m.weights.sum() - 16.0 * math.pi) < 1e-11 and m.weights.min() > 0
    assert m.weights.max() / m.weights.min() < 2.0
    per = body.Periphery(m)
    assert per.contains(np.array([[0.0, 0.0, 1.9]]))[0] and not per.contains(
        np.array([[0.0, 0.0, 2.1]]))[0]
