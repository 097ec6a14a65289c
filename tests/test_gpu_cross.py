"""Fiber <-> surface pairs evaluated once per pair (sf_cross.cu) against the
separate per-target sweeps (SF_CROSS=0), on the C4 confined aster (65,536
fiber points, 40,960-node periphery, centrosome) and a C2-sized aster."""

import numpy as np
import pytest

from paper_1602_05650_b200 import configs
from paper_1602_05650_b200.system import InteractionCache

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("which", ["c4", "c2"])
def test_cross_kernel_matches_separate_sweeps(cuda, which, monkeypatch):
    import torch
    st = configs.confined_aster() if which == "c4" else configs.aster(n_fibers=512, mesh_res=(16, 16))
    cache = InteractionCache(st)
    rng = np.random.default_rng(3)
    f = torch.as_tensor(rng.standard_normal((cache.fsrc.shape[0], 3)), device=cuda)
    q = torch.as_tensor(rng.standard_normal((cache.nss, 3)), device=cuda)
    w = torch.as_tensor(rng.standard_normal((len(st.particles), 6)), device=cuda)
    monkeypatch.setenv("SF_CROSS", "0")
    ref = cache.apply(f, q, w).cpu().numpy()
    monkeypatch.setenv("SF_CROSS", "1")
    got = cache.apply(f, q, w).cpu().numpy()
    again = cache.apply(f, q, w).cpu().numpy()
    assert np.array_equal(got, again)                      # deterministic
    fs, ps = cache.fiber_slice, slice(0, cache.fiber_slice.start)
    assert rel(got[fs], ref[fs]) < 1e-13
    assert rel(got[ps], ref[ps]) < 1e-13


def test_symmetric_subtracted_double_layer(cuda, monkeypatch):
    """On-surface subtracted double layer of the C4 periphery (40,960 nodes):
    symmetric evaluation vs the per-target sweep and the oracle
    (kernels.py:216-249)."""
    import torch
    from oracle import pairs
    from paper_1602_05650_b200 import body, kernels
    m = body.make_surface(body.sphere_shape(2.0), (40, 64))
    q = np.random.default_rng(4).standard_normal((m.n_nodes, 3))
    args = [torch.as_tensor(a, device=cuda) for a in (m.nodes, m.normals, m.weights, q)]
    pref = -3.0 / (4.0 * np.pi)
    monkeypatch.setenv("SF_SYMMETRIC", "0")
    ref = kernels.stresslet_sum_subtracted(*args, pref).cpu().numpy()
    monkeypatch.setenv("SF_SYMMETRIC", "1")
    got = kernels.stresslet_sum_subtracted(*args, pref).cpu().numpy()
    assert rel(got, ref) < 1e-13
    orc = pairs.stresslet_sum_subtracted(m.nodes, m.normals, m.weights, q, pref)   # ~1 s
    assert rel(got, orc) < 1e-12
