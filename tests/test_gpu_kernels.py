"""Parity of the sm_100a kernels (through the C ABI) with the reference.

Tolerances: FP64 path rel-L2 <= 1e-10 (north_star), asserted tighter where the
arithmetic allows; FP32-compute path <= 1e-5; integer outputs (`bad`) exact;
K_delta bitwise (explicitly rounded build).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import ops, pairs
from paper_1602_05650_b200 import kernels
from paper_1602_05650_b200.operator import FiberHIOperator

pytestmark = pytest.mark.gpu
rel = ops.rel_l2


def test_stokeslet_host_path(cuda):
    g = golden("pairs_small.npz")
    out, bad = kernels.stokeslet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], g["pref"])
    assert bad == int(g["stokeslet_bad"]) == 1
    assert rel(out, g["stokeslet"]) < 1e-14


def test_doublet_and_fused(cuda):
    g = golden("pairs_small.npz")
    out, bad = kernels.doublet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], g["pref"])
    assert bad == int(g["doublet_bad"])
    assert rel(out, g["doublet"]) < 1e-14
    c = np.full(g["src"].shape[0], 0.37)
    fused, bad = kernels.sbt_pair_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], c,
                                      g["pref"])
    assert bad == 1
    assert rel(fused, g["stokeslet"] + 0.37 * g["doublet"]) < 1e-14


def test_stresslet_and_surface_self_terms(cuda):
    g = golden("pairs_small.npz")
    out, bad = kernels.stresslet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["nrm"], g["qw"],
                                     g["spref"])
    assert bad == int(g["stresslet_bad"])
    assert rel(out, g["stresslet"]) < 1e-14
    sub = kernels.stresslet_sum_subtracted(g["mesh_nodes"], g["mesh_normals"], g["mesh_weights"],
                                           g["q"], g["spref"])
    assert rel(sub, g["subtracted"]) < 1e-13
    const = np.tile([0.4, -1.0, 2.0], (g["mesh_nodes"].shape[0], 1))
    zero = kernels.stresslet_sum_subtracted(g["mesh_nodes"], g["mesh_normals"],
                                            g["mesh_weights"], const, g["spref"])
    assert np.max(np.abs(zero)) == 0.0
    rs = kernels.stresslet_rowsum(g["mesh_nodes"], g["mesh_normals"], g["mesh_weights"],
                                  g["spref"])
    assert rel(rs, g["rowsum"]) < 1e-13


def test_kdelta_bitwise(cuda):
    g = golden("pairs_small.npz")
    K = kernels.kdelta_matrix(g["kd_X"], g["kd_s"], g["kd_sa"], g["kd_t"], g["kd_w"],
                              float(g["kd_delta"]), float(g["kd_pref"]))
    assert np.array_equal(K, g["kd_K"])


def test_group_exclusion_and_singular_counting(cuda):
    # test_kernels.py:139-147: the coincident own-group point is excluded, not bad
    src = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    f = np.array([[1.0, 0, 0], [0, 1.0, 0]])
    out, bad = kernels.stokeslet_sum(np.array([[0.0, 0, 0]]), np.array([0]), src,
                                     np.array([0, 1]), f, 1.0 / (8 * np.pi))
    assert bad == 0
    r = np.array([-1.0, 0, 0])
    expect = (f[1] / 1.0 + (r @ f[1]) * r) / (8 * np.pi) * (8 * np.pi) / (8 * np.pi)
    assert np.allclose(out[0], expect, rtol=1e-15, atol=0)
    # cross-group coincidence is counted (system.py:102-104 raises on it)
    out, bad = kernels.stokeslet_sum(src[:1], np.array([1]), src, np.array([0, 1]), f, 1.0)
    assert bad == 1


def test_empty_and_ungrouped(cuda):
    out, bad = kernels.stokeslet_sum(np.zeros((0, 3)), np.zeros(0, np.int64), np.ones((5, 3)),
                                     np.zeros(5, np.int64), np.ones((5, 3)), 1.0)
    assert out.shape == (0, 3) and bad == 0
    out, bad = kernels.stokeslet_sum(np.ones((4, 3)), None, np.zeros((0, 3)), None,
                                     np.zeros((0, 3)), 1.0)
    assert np.all(out == 0.0) and bad == 0
    rng = np.random.default_rng(5)
    t, s, f = rng.standard_normal((33, 3)), rng.standard_normal((71, 3)), rng.standard_normal((71, 3))
    ng_t, ng_s = kernels.no_groups(33), kernels.no_groups(71)
    a, _ = kernels.stokeslet_sum(t, ng_t, s, ng_s, f, 0.3)
    b, _ = kernels.stokeslet_sum(t, None, s, None, f, 0.3)
    ref, _ = pairs.stokeslet_sum(t, ng_t, s, ng_s, f, 0.3)
    assert np.array_equal(a, b) and rel(a, ref) < 1e-14


@pytest.mark.parametrize("nt,ns", [(1000, 200_000), (70_001, 70_001), (257, 129)])
def test_split_and_ragged_sizes_row_sampled(cuda, nt, ns):
    """Row-sampled oracle: any target subset reproduces its rows."""
    rng = np.random.default_rng(nt + ns)
    trg = rng.uniform(-10, 10, (nt, 3))
    src = rng.uniform(-10, 10, (ns, 3))
    sgrp = (np.arange(ns) // 64).astype(np.int64)
    tgrp = rng.integers(-1, ns // 64 + 1, nt).astype(np.int64)
    f = rng.standard_normal((ns, 3))
    c = rng.uniform(0, 1e-4, ns)
    out, bad = kernels.sbt_pair_sum(trg, tgrp, src, sgrp, f, c, 0.04)
    rows = rng.choice(nt, size=min(nt, 300), replace=False)
    st, _ = pairs.stokeslet_sum(trg[rows], tgrp[rows], src, sgrp, f, 0.04)
    db, _ = pairs.doublet_sum(trg[rows], tgrp[rows], src, sgrp, c[:, None] * f, 0.04)
    assert bad == 0
    assert rel(out[rows], st + db) < 1e-13


def test_device_path_is_deterministic(cuda):
    import torch
    rng = np.random.default_rng(8)
    n = 50_000
    x = torch.as_tensor(rng.uniform(-5, 5, (n, 3)), device=cuda)
    g = torch.as_tensor((np.arange(n) // 32).astype(np.int64), device=cuda)
    f = torch.as_tensor(rng.standard_normal((n, 3)), device=cuda)
    a, _ = kernels.stokeslet_sum(x, g, x, g, f, 1.0)
    b, _ = kernels.stokeslet_sum(x, g, x, g, f, 1.0)
    assert torch.equal(a, b)
    host, _ = kernels.stokeslet_sum(x.cpu().numpy(), g.cpu().numpy(), x.cpu().numpy(),
                                    g.cpu().numpy(), f.cpu().numpy(), 1.0)
    assert np.array_equal(a.cpu().numpy(), host)


def test_fp32c_variant(cuda):
    g = golden("c1_clean.npz")
    X = g["X"].reshape(-1, 3)
    grp = np.repeat(np.arange(g["X"].shape[0]), g["X"].shape[1]).astype(np.int64)
    w = g["weights"].reshape(-1)
    c = np.repeat((float(g["eps"]) * g["L"]) ** 2 / 2.0, g["X"].shape[1])
    f = w[:, None] * g["forces"].reshape(-1, 3)
    pref = 1.0 / (8 * np.pi)
    out64, _ = kernels.sbt_pair_sum(X, grp, X, grp, f, c, pref, mode=kernels.SF_MODE_FP64)
    out32, _ = kernels.sbt_pair_sum(X, grp, X, grp, f, c, pref, mode=kernels.SF_MODE_FP32C)
    assert rel(out64, g["u_nl"]) < 1e-12
    assert rel(out32, g["u_nl"]) < 1e-5


@pytest.mark.parametrize("name", ["c1_near.npz", "c1_clean.npz"])
def test_fiber_operator_c1(cuda, name):
    g = golden(name)
    near = [(int(t), int(l), W) for t, l, W in zip(g["near_t"], g["near_l"], g["near_W"])]
    op = FiberHIOperator(g["X"], float(g["eps"]), float(g["mu"]), near=near)
    u_nl, u_self = op.apply(g["forces"])
    op.check_bad()
    assert rel(u_nl.cpu().numpy(), g["u_nl"]) < 1e-12
    assert rel(u_self.cpu().numpy(), g["u_self"]) < 1e-12
    # K from device-computed geometry: equal to rounding (bitwise given the
    # reference's own geometry, test_kdelta_bitwise)
    K = op.K[:2].cpu().numpy()
    assert np.abs(K - g["K"]).max() <= 1e-13 * np.abs(g["K"]).max()
    assert np.abs(op.s.cpu().numpy() - g["s"]).max() < 1e-14
    assert np.abs(op.tang.cpu().numpy() - g["tangents"]).max() < 1e-12
    assert np.abs(op.delta.cpu().numpy() - g["delta"]).max() < 1e-16


def _cloud_operator_inputs(nf=200, n=64, seed=3):
    from paper_1602_05650_b200 import configs
    cl = configs.fiber_cloud(nf, n - 1, eps=5e-3, E=1e-2, region="ball", size=4.0, seed=seed,
                             clear=configs.clean_clear(n - 1), check="node", perturb=1e-2)
    return cl, configs.forces(cl, seed=seed + 1)


@pytest.mark.parametrize("nf,n", [(200, 64), (333, 32), (401, 24)])
def test_symmetric_matches_direct_and_oracle(cuda, nf, n):
    """The symmetric (both directions per pair geometry) evaluation equals the
    per-target direct sum to rounding, is bitwise reproducible, and matches
    the oracle on sampled rows; sizes exercise partial units and fibers that
    do not divide the 32-point slabs."""
    from paper_1602_05650_b200._native import SF_MODE_FP64, SF_MODE_FP64_DIRECT
    cl, F = _cloud_operator_inputs(nf, n)
    assert cl.n_points >= 8192
    sym = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64)
    direct = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64_DIRECT)
    a, _ = sym.apply(F, self_terms=False)
    b, _ = sym.apply(F, self_terms=False)
    c, _ = direct.apply(F, self_terms=False)
    sym.check_bad()
    a, b, c = a.cpu().numpy(), b.cpu().numpy(), c.cpu().numpy()
    assert np.array_equal(a, b)
    assert rel(a, c) < 1e-13
    rng = np.random.default_rng(0)
    rows = rng.choice(cl.n_points, 200, replace=False)
    X = cl.X.reshape(-1, 3)
    grp = np.repeat(np.arange(cl.n_fibers), cl.n_nodes)
    w = sym.wnode.cpu().numpy().reshape(-1)
    L = sym.L.cpu().numpy()
    s = w[:, None] * F.reshape(-1, 3)
    cc = np.repeat((cl.eps * L) ** 2 / 2.0, cl.n_nodes)
    pref = 1.0 / (8.0 * np.pi)
    st, _ = pairs.stokeslet_sum(X[rows], grp[rows], X, grp, s, pref)
    db, _ = pairs.doublet_sum(X[rows], grp[rows], X, grp, cc[:, None] * s, pref)
    assert rel(a[rows], st + db) < 1e-13


def test_symmetric_counts_coincident_pairs(cuda):
    from paper_1602_05650_b200._native import SF_MODE_FP64
    cl, F = _cloud_operator_inputs(160, 64)
    X = cl.X.copy()
    X[7, 10] = X[90, 33]          # cross-fiber coincidence: 2 bad ordered pairs
    op = FiberHIOperator(X, cl.eps, mode=SF_MODE_FP64)
    op.apply(F, self_terms=False)
    assert int(op.bad.item()) == 2
    with pytest.raises(kernels.SingularEvaluationError):
        op.check_bad()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_symmetric_task_shards_sum_to_single_gpu(cuda, world):
    """Multi-GPU symmetric form emulated on one GPU: the ranks' task shares,
    each contributing to every point, sum to the single-GPU result."""
    import torch
    from paper_1602_05650_b200._native import SF_MODE_FP64
    cl, F = _cloud_operator_inputs(200, 64)
    op = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64)
    one, _ = op.apply(F, self_terms=False)
    total = torch.zeros_like(one)
    for r in range(world):
        total += op.symmetric_partial(F, rank=r, world=world)
    assert rel(total.cpu().numpy(), one.cpu().numpy()) < 1e-14


@pytest.mark.parametrize("nf,n", [(200, 64), (333, 32), (401, 24)])
def test_symmetric_fp32c_variant(cuda, nf, n):
    """FP32-compute / FP64-accumulate symmetric evaluation within 1e-5 of FP64
    (slab-relative FP32 positions); the sizes give partial units, padding i
    lanes and j slabs, and fibers that straddle slabs."""
    from paper_1602_05650_b200._native import SF_MODE_FP32C, SF_MODE_FP64
    cl, F = _cloud_operator_inputs(nf, n)
    a, _ = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64).apply(F, self_terms=False)
    op32 = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP32C)
    assert op32.symmetric
    b, _ = op32.apply(F, self_terms=False)
    c, _ = op32.apply(F, self_terms=False)
    assert torch_equal(b, c)
    e = rel(b.cpu().numpy(), a.cpu().numpy())
    assert e < 1e-5, e


def test_symmetric_fp32c_counts_coincident_pairs(cuda):
    from paper_1602_05650_b200._native import SF_MODE_FP32C
    cl, F = _cloud_operator_inputs(160, 64)
    X = cl.X.copy()
    X[7, 10] = X[90, 33]
    op = FiberHIOperator(X, cl.eps, mode=SF_MODE_FP32C)
    u, _ = op.apply(F, self_terms=False)
    assert int(op.bad.item()) == 2
    assert np.isfinite(u.cpu().numpy()).all()


def torch_equal(x, y):
    import torch
    return bool(torch.equal(x, y))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_operator_ranks_match_single_gpu(cuda, world):
    """The multi-GPU operator flow of dist.ShardedHIOperator emulated on one
    GPU: every rank's symmetric partial for all points, summed (the
    reduce-scatter), then each rank's near + self terms for its own targets,
    with the all-gathered (nf, n, 3) force array as the dist layer passes it."""
    import torch
    from paper_1602_05650_b200._native import SF_MODE_FP64
    cl, F = _cloud_operator_inputs(200, 64)
    Fd = torch.as_tensor(F, device=cuda).reshape(cl.X.shape[0], cl.X.shape[1], 3)
    one = FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64)
    u1, s1 = one.apply(Fd)
    ops = [FiberHIOperator(cl.X, cl.eps, mode=SF_MODE_FP64, shard=(r, world)) for r in range(world)]
    assert all(op.symmetric_shard for op in ops)
    total = sum(op.symmetric_partial(Fd) for op in ops)
    for op in ops:
        lo, hi = op.f0 * op.n, (op.f0 + op.nown) * op.n
        u, s = op.finish_own(total[lo:hi].clone(), Fd)
        assert rel(u.cpu().numpy(), u1[lo:hi].cpu().numpy()) < 1e-13
        assert torch.equal(s, s1[lo:hi])
