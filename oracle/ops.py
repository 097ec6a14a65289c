"""ORACLE (test infrastructure only): numpy restatement of the reference's
fiber/surface operators on the HI-operator path.

Each function cites the reference lines it restates
(/root/reference/pkg/src/slenderflow/...).  Pair sums go through the C
restatement in oracle.pairs, in the same two-pass structure the reference
uses (Stokeslet pass, then doublet pass, system.py:656-671).
"""

import math

import numpy as np
from numpy.polynomial import chebyshev as npc
from scipy.fft import dct

from . import pairs

# ------------------------------------------------------------ spectral.py ----


def cheb_nodes(p):
    """spectral.py:24-34."""
    a = np.cos(np.arange(p + 1) * np.pi / p)
    return 0.5 * (a - a[::-1])


def cheb_transform(v):
    """spectral.py:37-50 (type-I DCT)."""
    v = np.asarray(v, dtype=float)
    c = dct(v, type=1) / (v.size - 1)
    c[0] *= 0.5
    c[-1] *= 0.5
    return c


class Grid:
    """spectral.py:99-136: nodes, Clenshaw-Curtis weights, dense D."""

    def __init__(self, p):
        self.p = p
        self.nodes = cheb_nodes(p)
        k = np.arange(p + 1)
        mu = np.zeros(p + 1)
        ev = k % 2 == 0
        mu[ev] = 2.0 / (1.0 - k[ev].astype(float) ** 2)
        Cm = np.empty((p + 1, p + 1))
        for j in range(p + 1):
            e = np.zeros(p + 1)
            e[j] = 1.0
            Cm[:, j] = cheb_transform(e)
        self.weights = mu @ Cm
        self.D = np.empty((p + 1, p + 1))
        for j in range(p + 1):
            e = np.zeros(p + 1)
            e[j] = 1.0
            self.D[:, j] = npc.chebval(self.nodes, npc.chebder(cheb_transform(e)))


_GRIDS = {}


def grid(p):
    if p not in _GRIDS:
        _GRIDS[p] = Grid(p)
    return _GRIDS[p]


def geometry(X):
    """spectral.py:139-154 + fiber.py:133-147 for one fiber (n,3)."""
    g = grid(X.shape[0] - 1)
    Xa = g.D @ X
    s_alpha = np.sqrt((Xa * Xa).sum(axis=1))
    anti = npc.chebint(cheb_transform(s_alpha))
    s = npc.chebval(g.nodes, anti) - npc.chebval(-1.0, anti)
    L = float(s[0])
    return dict(s=s, s_alpha=s_alpha, L=L, tangents=Xa / s_alpha[:, None],
                weights=g.weights * s_alpha, delta=0.01 * L)


# --------------------------------------------------------------- fiber.py ----


def local_mobility_apply(tangents, eps, f, mu):
    """fiber.py:244-250."""
    c_log = -math.log(eps ** 2 * math.e) / (8.0 * np.pi * mu)
    c_two = 2.0 / (8.0 * np.pi * mu)
    ft = (f * tangents).sum(axis=1)[:, None] * tangents
    return c_log * (f + ft) + c_two * (f - ft)


def kdelta_matrix(X, geo, mu):
    """fiber.py:213-222 -> kernels.py:284-334 (C restatement)."""
    g = grid(X.shape[0] - 1)
    return pairs.kdelta_matrix(X, geo["s"], geo["s_alpha"], geo["tangents"], g.weights,
                               geo["delta"], 1.0 / (8.0 * np.pi * mu))


# -------------------------------------------------------------- system.py ----


def fiber_operator(X, forces, eps, mu=1.0, near=(), include_doublet=True):
    """The C1-form operator: fiber part of complementary_velocities
    (system.py:623-709, targets = sources = fiber nodes, groups = fiber ids)
    plus the per-fiber self terms M f + K f (fiber.py:244-258).

    X, forces: (nf, n, 3); eps: scalar or (nf,); near: iterable of (t, l, W).
    Returns (u_nl (N,3), u_self (N,3)).
    """
    nf, n, _ = X.shape
    eps = np.broadcast_to(np.asarray(eps, dtype=float), (nf,))
    geos = [geometry(X[m]) for m in range(nf)]
    src = X.reshape(-1, 3)
    grp = np.repeat(np.arange(nf, dtype=np.int64), n)
    w = np.concatenate([g["weights"] for g in geos])
    f = forces.reshape(-1, 3)
    pref = 1.0 / (8.0 * np.pi * mu)
    strengths = w[:, None] * f                                   # system.py:657-658
    u, bad = pairs.stokeslet_sum(src, grp, src, grp, strengths, pref)
    if bad:
        raise ValueError("a target coincides with a source outside its own group")
    if include_doublet:
        c = np.repeat([(eps[m] * geos[m]["L"]) ** 2 / 2.0 for m in range(nf)], n)
        out, bad = pairs.doublet_sum(src, grp, src, grp, c[:, None] * strengths, pref)
        if bad:
            raise ValueError("a target coincides with another fiber's node")
        u = u + out
    for t, l, W in near:                                         # system.py:702-707
        u[t] += W @ forces[l].ravel()
    u_self = np.concatenate([
        local_mobility_apply(geos[m]["tangents"], eps[m], forces[m], mu)
        + (kdelta_matrix(X[m], geos[m], mu) @ forces[m].ravel()).reshape(-1, 3)
        for m in range(nf)])
    return u, u_self


def rel_l2(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
