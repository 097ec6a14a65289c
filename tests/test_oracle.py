"""The oracle restatement is pinned to the reference's own outputs.

Golden vectors were produced by running /root/reference's slenderflow on the
same seeded inputs (tests/golden/make_golden.py).  The C restatement keeps
the reference's operation order and unfused arithmetic, so pair sums and
K_delta must match BITWISE; numpy-level compositions within 1e-13.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import ops, pairs


def test_stokeslet_sum_bitwise():
    g = golden("pairs_small.npz")
    out, bad = pairs.stokeslet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], g["pref"])
    assert bad == int(g["stokeslet_bad"]) == 1
    assert np.array_equal(out, g["stokeslet"])


def test_doublet_sum_bitwise():
    g = golden("pairs_small.npz")
    out, bad = pairs.doublet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], g["pref"])
    assert bad == int(g["doublet_bad"])
    assert np.array_equal(out, g["doublet"])


def test_stresslet_sum_bitwise():
    g = golden("pairs_small.npz")
    out, bad = pairs.stresslet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["nrm"], g["qw"],
                                   g["spref"])
    assert bad == int(g["stresslet_bad"])
    assert np.array_equal(out, g["stresslet"])


def test_surface_self_terms_bitwise():
    g = golden("pairs_small.npz")
    sub = pairs.stresslet_sum_subtracted(g["mesh_nodes"], g["mesh_normals"], g["mesh_weights"],
                                         g["q"], g["spref"])
    assert np.array_equal(sub, g["subtracted"])
    rs = pairs.stresslet_rowsum(g["mesh_nodes"], g["mesh_normals"], g["mesh_weights"], g["spref"])
    assert np.array_equal(rs, g["rowsum"])
    const = np.tile([0.4, -1.0, 2.0], (g["mesh_nodes"].shape[0], 1))
    zero = pairs.stresslet_sum_subtracted(g["mesh_nodes"], g["mesh_normals"], g["mesh_weights"],
                                          const, g["spref"])
    assert np.max(np.abs(zero)) == 0.0 and np.array_equal(zero, g["subtracted_const"])


def test_kdelta_bitwise():
    g = golden("pairs_small.npz")
    K = pairs.kdelta_matrix(g["kd_X"], g["kd_s"], g["kd_sa"], g["kd_t"], g["kd_w"],
                            float(g["kd_delta"]), float(g["kd_pref"]))
    assert np.array_equal(K, g["kd_K"])


def test_thread_count_independence():
    g = golden("pairs_small.npz")
    n0 = pairs.num_threads()
    try:
        pairs.set_num_threads(1)
        a, _ = pairs.stokeslet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], g["pref"])
        pairs.set_num_threads(max(n0, 3))
        b, _ = pairs.stokeslet_sum(g["trg"], g["tgrp"], g["src"], g["sgrp"], g["f"], g["pref"])
    finally:
        pairs.set_num_threads(n0)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["c1_near.npz", "c1_clean.npz"])
def test_operator_matches_reference(name):
    g = golden(name)
    X = g["X"]
    near = [(int(t), int(l), W) for t, l, W in zip(g["near_t"], g["near_l"], g["near_W"])]
    u_nl, u_self = ops.fiber_operator(X, g["forces"], float(g["eps"]), float(g["mu"]), near)
    assert ops.rel_l2(u_nl, g["u_nl"]) < 1e-13
    assert ops.rel_l2(u_self, g["u_self"]) < 1e-13
    geo = ops.geometry(X[0])
    assert np.array_equal(geo["s_alpha"], g["s_alpha"][0])
    assert np.abs(geo["s"] - g["s"][0]).max() < 1e-15
    K0 = ops.kdelta_matrix(X[0], geo, float(g["mu"]))
    assert np.abs(K0 - g["K"][0]).max() <= 1e-13 * np.abs(g["K"][0]).max()


def test_c1_near_fixture_has_near_pairs():
    g = golden("c1_near.npz")
    assert g["near_t"].size > 0
    assert golden("c1_clean.npz")["near_t"].size == 0
