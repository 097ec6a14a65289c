"""Bounded partial storage of the symmetric fiber-pair kernel (sf_sym.cu):
the tasks run in waves of task rows, each wave's partials in a compact
buffer, added to the running per-point sums in slot order.  The result is
bitwise independent of the wave budget and of the number of wave streams,
and the scratch the library holds stays within the budget."""

import numpy as np
import pytest
import torch

from paper_1602_05650_b200 import _native, configs
from paper_1602_05650_b200.operator import FiberHIOperator

pytestmark = pytest.mark.gpu


@pytest.fixture
def waves_reset():
    yield
    _native.load().sf_sym_set_waves(0, 0)


def _apply(op, f):
    u, _ = op.apply(f, self_terms=False)
    torch.cuda.synchronize()
    return u.clone()


@pytest.mark.parametrize("mode", [_native.SF_MODE_FP64, _native.SF_MODE_FP32C])
def test_waves_are_bitwise_independent_of_budget(cuda, waves_reset, mode):
    cl = configs.make("c3_scaled", seed=1, n_fibers=1024, size=6.3)        # N = 65,536
    f = configs.forces(cl, seed=2)
    lib = _native.load()
    op = FiberHIOperator(cl.X, cl.eps, device=cuda, mode=mode)
    assert op.symmetric
    lib.sf_sym_set_waves(1 << 40, 1)                 # one wave
    ref = _apply(op, f)
    one = lib.sf_sym_launch_count(op.N, op.n, mode, 0, 1)
    for budget, streams in ((1, 1), (1, 3), (4 << 20, 2), (16 << 20, 3)):
        lib.sf_sym_set_waves(budget, streams)        # 1 byte: one task row per wave
        assert lib.sf_sym_launch_count(op.N, op.n, mode, 0, 1) > one
        assert torch.equal(_apply(op, f), ref), (budget, streams)


def test_waves_match_direct_and_oracle_rows(cuda, waves_reset):
    """Many waves (one row each) still equal the per-target direct kernel to
    rounding, and the oracle on sampled rows."""
    from oracle import pairs
    cl = configs.make("c3_scaled", seed=3, n_fibers=512)
    f = configs.forces(cl, seed=4)
    _native.load().sf_sym_set_waves(1, 3)
    sym = FiberHIOperator(cl.X, cl.eps, device=cuda)
    direct = FiberHIOperator(cl.X, cl.eps, device=cuda, mode=_native.SF_MODE_FP64_DIRECT)
    a, b = _apply(sym, f), _apply(direct, f)
    assert float((a - b).norm() / b.norm()) < 1e-13
    from oracle import ops
    X = cl.X.reshape(-1, 3)
    n = cl.n_nodes
    grp = np.repeat(np.arange(cl.n_fibers, dtype=np.int64), n)
    geos = [ops.geometry(cl.X[m]) for m in range(cl.n_fibers)]
    w = np.concatenate([g["weights"] for g in geos])
    s = w[:, None] * f.reshape(-1, 3)
    c = np.repeat([(cl.eps * g["L"]) ** 2 / 2.0 for g in geos], n)
    rows = np.random.default_rng(0).choice(X.shape[0], 64, replace=False)
    pref = 1.0 / (8.0 * np.pi)
    u1, _ = pairs.stokeslet_sum(X[rows], grp[rows], X, grp, s, pref)
    u2, _ = pairs.doublet_sum(X[rows], grp[rows], X, grp, c[:, None] * s, pref)
    got = a.cpu().numpy()[rows]
    assert np.linalg.norm(got - (u1 + u2)) / np.linalg.norm(u1 + u2) < 1e-12


def test_c5_scratch_is_bounded(cuda, waves_reset):
    """C5 (1,048,576 points): the library's scratch after one evaluation stays
    near 2 x 192 MB of wave buffers plus the packed sources and sums (the
    unbounded G x N x 3 slot buffer was 8.6 GB)."""
    lib = _native.load()
    cl = configs.make("c5", seed=0)
    f = configs.forces(cl, seed=1)
    op = FiberHIOperator(cl.X, cl.eps, device=cuda)
    lib.sf_workspace_release()             # scratch other tests' calls left behind
    assert lib.sf_workspace_bytes() == 0
    _apply(op, f)
    held = lib.sf_workspace_bytes()
    assert held < 1.0e9, held


def test_twice_c5_fits_one_gpu(cuda, waves_reset):
    """2 x C5 (32,768 fibers x 64 = 2,097,152 points) on ONE GPU: the wave
    buffers keep the scratch bounded (the round-1 slot buffer would have
    needed G N 3 doubles = 34 GB), and sampled rows match the oracle."""
    from oracle import pairs
    lib = _native.load()
    cl = configs.make("c5", seed=2, n_fibers=32768, size=20.0 * 2.0 ** (1.0 / 3.0))
    f = configs.forces(cl, seed=3)
    op = FiberHIOperator(cl.X, cl.eps, device=cuda)
    lib.sf_workspace_release()
    u = _apply(op, f)
    assert lib.sf_workspace_bytes() < 1.5e9
    X = cl.X.reshape(-1, 3)
    grp = np.repeat(np.arange(cl.n_fibers, dtype=np.int64), cl.n_nodes)
    s = op.wnode.cpu().numpy().reshape(-1)[:, None] * f.reshape(-1, 3)
    c = np.repeat((cl.eps * op.L.cpu().numpy()) ** 2 / 2.0, cl.n_nodes)
    rows = np.random.default_rng(4).choice(X.shape[0], 16, replace=False)
    pref = 1.0 / (8.0 * np.pi)
    u1, _ = pairs.stokeslet_sum(X[rows], grp[rows], X, grp, s, pref)
    u2, _ = pairs.doublet_sum(X[rows], grp[rows], X, grp, c[:, None] * s, pref)
    got = u.cpu().numpy()[rows]
    assert np.linalg.norm(got - (u1 + u2)) / np.linalg.norm(u1 + u2) < 1e-12
