"""Parity at BASELINE's full sizes: the C5 (1,048,576 points)
and C3 (262,144 points) operators against the oracle on sampled target rows
(each row is the reference's serial source loop, so a row subset is exact),
plus size-independent properties on the whole vector: symmetric vs direct
evaluation, FP32c vs FP64 (tolerance 1e-5), linearity, bitwise
reproducibility."""

import numpy as np
import pytest

from oracle import pairs
from paper_1602_05650_b200 import configs
from paper_1602_05650_b200.operator import FiberHIOperator

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module", params=["c5", "c3"])
def big(request):
    cl = configs.make(request.param, seed=0)
    return request.param, cl, configs.forces(cl, seed=1)


def oracle_rows(cl, op, F, rows):
    X = cl.X.reshape(-1, 3)
    grp = np.repeat(np.arange(cl.n_fibers), cl.n_nodes)
    s = op.wnode.cpu().numpy().reshape(-1)[:, None] * F.reshape(-1, 3)
    cc = np.repeat((cl.eps * op.L.cpu().numpy()) ** 2 / 2.0, cl.n_nodes)
    pref = 1.0 / (8.0 * np.pi)
    st, _ = pairs.stokeslet_sum(X[rows], grp[rows], X, grp, s, pref)
    db, _ = pairs.doublet_sum(X[rows], grp[rows], X, grp, cc[:, None] * s, pref)
    return st + db


def test_full_size_operator_parity(cuda, big):
    import torch
    from paper_1602_05650_b200._native import SF_MODE_FP32C, SF_MODE_FP64, SF_MODE_FP64_DIRECT
    name, cl, F = big
    Fd = torch.as_tensor(F, device=cuda)
    op = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64)
    assert op.symmetric
    a = op.apply(Fd, self_terms=False)[0].cpu().numpy()
    a2 = op.apply(Fd, self_terms=False)[0].cpu().numpy()
    op.check_bad()
    assert np.array_equal(a, a2)                                   # reproducible
    rows = np.random.default_rng(7).choice(cl.n_points, 192, replace=False)
    assert rel(a[rows], oracle_rows(cl, op, F, rows)) < 1e-12      # FP64 vs oracle
    d = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64_DIRECT).apply(Fd, self_terms=False)[0]
    assert rel(a, d.cpu().numpy()) < 1e-13                        # two kernels, one sum
    del d
    b = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP32C).apply(Fd, self_terms=False)[0]
    assert rel(b.cpu().numpy(), a) < 1e-5                         # FP32c tolerance
    # linearity (size independent): A(F + 2G) = A F + 2 A G
    G = torch.as_tensor(configs.forces(cl, seed=5), device=cuda)
    lin = op.apply(Fd + 2.0 * G, self_terms=False)[0].cpu().numpy()
    ag = op.apply(G, self_terms=False)[0].cpu().numpy()
    assert rel(lin, a + 2.0 * ag) < 1e-12


def test_full_size_reference_api_with_near_maps(cuda, big):
    """complementary_velocities (the reference's signature, host arrays in and
    out) at full size equals the batched operator given the same near maps;
    rows with near maps are the oracle's pair sum plus W . f of the source
    fiber (system.py:702-707)."""
    import torch
    from paper_1602_05650_b200 import system
    from paper_1602_05650_b200.fiber import Fiber
    name, cl, F = big
    st = system.SystemState([Fiber(X, eps=cl.eps, E=cl.E) for X in cl.X])
    cache = system.InteractionCache(st)
    ua = np.concatenate(system.complementary_velocities(st, fiber_forces=list(F), cache=cache).fibers)
    op = FiberHIOperator(cl.X, cl.eps, near=cache.near_fiber)
    ub = op.apply(torch.as_tensor(F, device=cuda), self_terms=False)[0].cpu().numpy()
    assert rel(ua, ub) < 1e-14
    if cache.near_fiber:                      # C5: 2 targets inside a near shell
        rows = np.array(sorted({t for t, _, _ in cache.near_fiber}))
        corr = np.zeros((rows.size, 3))
        for t, l, W in cache.near_fiber:
            W = W.cpu().numpy() if torch.is_tensor(W) else np.asarray(W)
            corr[np.searchsorted(rows, t)] += W.reshape(3, -1) @ F[l].reshape(-1)
        assert rel(ua[rows], oracle_rows(cl, op, F, rows) + corr) < 1e-12


@pytest.mark.parametrize("name", ["c4", "c2"])
def test_aster_full_size_rows_match_oracle(cuda, name):
    """BASELINE configs 4 (2,048 fibers x 32, 40,960-node periphery,
    centrosome, ~116k near maps) and 2 (1,024-fiber aster on an (8,8)
    particle) at full size: complementary_velocities on sampled target rows
    against the reference's composition (system.py:653-707) restated with
    the oracle's pair sums, the completion flow and the cache's near-field
    maps.  Rows of every kind (particle, periphery, fibers, near-map
    targets) are sampled."""
    import torch
    from paper_1602_05650_b200 import system
    st = configs.confined_aster() if name == "c4" else configs.aster(n_fibers=1024)
    cache = system.InteractionCache(st)
    rng = np.random.default_rng(11)
    f_list = [rng.standard_normal((fb.n_nodes, 3)) for fb in st.fibers]
    q1 = rng.standard_normal((st.particles[0].mesh.n_nodes, 3))
    q0 = (rng.standard_normal((st.periphery.mesh.n_nodes, 3)) if st.periphery is not None
          else None)
    F, L = rng.standard_normal(3), rng.standard_normal(3)
    res = system.complementary_velocities(st, periphery_density=q0, particle_densities=[q1],
                                          fiber_forces=f_list, particle_wrenches=[(F, L)],
                                          cache=cache)
    u = np.concatenate([res.particles[0]] + ([res.periphery] if q0 is not None else [])
                       + list(res.fibers))
    trg, tgrp = cache.targets, cache.target_groups
    near_t = np.array(sorted({t for t, _, _ in cache.near_fiber}), dtype=np.int64)
    picks = [rng.choice(cache.particle_slices[0].stop, 24, replace=False),
             cache.fiber_slice.start + rng.choice(cache.fiber_slice.stop - cache.fiber_slice.start,
                                                  96, replace=False)]
    if q0 is not None:
        picks.append(cache.periphery_slice.start +
                     rng.choice(st.periphery.mesh.n_nodes, 48, replace=False))
    if near_t.size:
        picks.append(rng.choice(near_t, min(48, near_t.size), replace=False))
    rows = np.unique(np.concatenate(picks))
    mu = st.mu
    src = np.concatenate([fb.X for fb in st.fibers])
    sgrp = np.repeat(np.arange(len(st.fibers), dtype=np.int64), [fb.n_nodes for fb in st.fibers])
    w = np.concatenate(cache.fiber_weights)
    f = np.concatenate(f_list)
    c = np.repeat(cache.doublet_coeffs, [fb.n_nodes for fb in st.fibers])
    pref = 1.0 / (8.0 * np.pi * mu)
    ref, _ = pairs.stokeslet_sum(trg[rows], tgrp[rows], src, sgrp, w[:, None] * f, pref)
    ref += pairs.doublet_sum(trg[rows], tgrp[rows], src, sgrp, (c * w)[:, None] * f, pref)[0]
    meshes = [m for m, _, _ in cache.surfaces]
    qs = [q0 if isp else q1 for _, _, isp in cache.surfaces]
    qw = np.concatenate([q * m.weights[:, None] for q, m in zip(qs, meshes)])
    ref += pairs.stresslet_sum(trg[rows], tgrp[rows], cache.surface_sources, cache.surface_groups,
                               cache.surface_normals, qw, -3.0 / (4.0 * np.pi * mu))[0]
    part = st.particles[0]
    mask = tgrp[rows] != len(st.fibers)
    r = trg[rows][mask] - part.center
    d = np.linalg.norm(r, axis=1)
    ref[mask] += pref * (F[None, :] / d[:, None] + ((r @ F) / d ** 3)[:, None] * r)
    ref[mask] += pref * np.cross(L[None, :], r) / (d ** 3)[:, None]
    pos = {t: k for k, t in enumerate(rows)}
    for t, l, W in cache.near_fiber:
        if t in pos:
            W = W.cpu().numpy() if torch.is_tensor(W) else np.asarray(W)
            ref[pos[t]] += W.reshape(3, -1) @ f_list[l].ravel()
    for t, si, W in cache.near_surface:
        if t in pos:
            W = W.cpu().numpy() if torch.is_tensor(W) else np.asarray(W)
            ref[pos[t]] += W.reshape(3, -1) @ qs[si].ravel()
    assert rel(u[rows], ref) < 1e-12


def test_full_size_self_terms_match_oracle(cuda, big):
    """u_self = M f + K_delta f (fiber.py:244-258), the local part of the bench
    step, at full C5 / C3 size: 48 sampled fibers against the oracle's
    per-fiber local mobility and K_delta matrix (oracle/ops.py)."""
    import torch

    from oracle import ops
    name, cl, F = big
    op = FiberHIOperator(cl.X, cl.eps)
    _, u_self = op.apply(torch.as_tensor(F, device=cuda), self_terms=True)
    u_self = u_self.cpu().numpy().reshape(cl.n_fibers, cl.n_nodes, 3)
    fibs = np.random.default_rng(9).choice(cl.n_fibers, 48, replace=False)
    errs = []
    for m in fibs:
        geo = ops.geometry(cl.X[m])
        ref = ops.local_mobility_apply(geo["tangents"], cl.eps, F[m], 1.0) + \
            (ops.kdelta_matrix(cl.X[m], geo, 1.0) @ F[m].ravel()).reshape(-1, 3)
        errs.append(rel(u_self[m], ref))
    print(f"{name} u_self per-fiber rel L2: max {max(errs):.2e}, median {np.median(errs):.2e}")
    assert max(errs) < 1e-10          # north_star operator tolerance
