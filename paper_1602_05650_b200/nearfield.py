"""Near-field correction maps for targets inside a fiber's near shell.

Host construction of the small linear maps W (3 x 3n) that replace the plain
collocation sum for targets closer than 1.5 L/p to another fiber, following
the reference's algorithm (fiber.py:453-575, system.py:564-586): nearest
centreline point by refined sampling plus golden-section search, adaptive
bisection into 10-point Gauss-Legendre panels until each is shorter than its
distance to the target, barycentric resampling of the nodal density, and a
smoothstep blend back to the plain sum near the shell boundary.  The maps are
built once per geometry and applied on the device every matvec
(sf_near_apply); moving their construction to the device is the next step
(SURVEY.md §8f rank 1).
"""

import math

import numpy as np
from numpy.polynomial import chebyshev as C

from . import spectral
from .fiber import InsideFiberError

NEAR_SHELL_FACTOR = 1.5
_GL10_X, _GL10_W = np.polynomial.legendre.leggauss(10)


def _coeffs(values):
    return spectral.values_to_coeffs(values)


def nearest_centerline_point(fib, target):
    """(alpha, point, distance) of the closest centreline point (fiber.py:453-481)."""
    target = np.asarray(target, dtype=float)
    cx = [_coeffs(fib.X[:, c]) for c in range(3)]
    al = np.cos(np.linspace(0.0, np.pi, 8 * fib.p + 1))
    Xf = np.stack([C.chebval(al, c) for c in cx], axis=1)
    i0 = int(((Xf - target) ** 2).sum(axis=1).argmin())
    lo = al[min(i0 + 1, al.size - 1)]
    hi = al[max(i0 - 1, 0)]

    def d2_at(a):
        x = np.array([C.chebval(a, c) for c in cx])
        return ((x - target) ** 2).sum()

    for _ in range(50):
        m1 = lo + 0.382 * (hi - lo)
        m2 = lo + 0.618 * (hi - lo)
        if d2_at(m1) < d2_at(m2):
            hi = m2
        else:
            lo = m1
    a0 = 0.5 * (lo + hi)
    x0 = np.array([C.chebval(a0, c) for c in cx])
    return a0, x0, float(np.linalg.norm(target - x0))


def _bary_rows(alphas, p):
    nodes = spectral.cheb_nodes(p)
    alphas = np.atleast_1d(np.asarray(alphas, dtype=float))
    w = np.ones(p + 1)
    w[1::2] = -1.0
    w[0] *= 0.5
    w[-1] *= 0.5
    d = alphas[:, None] - nodes[None, :]
    hit = np.abs(d) < 1e-14
    t = w[None, :] / np.where(hit, 1.0, d)
    rows = t / t.sum(axis=1)[:, None]
    on = hit.any(axis=1)
    rows[on] = hit[on].astype(float)
    return rows


def _kernel_blocks(r, include_doublet, coeff):
    d2 = (r * r).sum(axis=1)
    d = np.sqrt(d2)
    eye = np.eye(3)
    rr = r[:, :, None] * r[:, None, :]
    K = eye[None] / d[:, None, None] + rr / (d2 * d)[:, None, None]
    if include_doublet:
        K += coeff * (eye[None] / (d2 * d)[:, None, None] - 3.0 * rr / (d2 * d2 * d)[:, None, None])
    return K


def plain_fiber_weights(fib, target, mu, include_doublet=False):
    """Collocation-sum linear map (fiber.py:568-575)."""
    target = np.asarray(target, dtype=float)
    coeff = (fib.eps * fib.L) ** 2 / 2.0
    K = _kernel_blocks(target[None, :] - fib.X, include_doublet, coeff)
    W = np.einsum("j,jab->ajb", fib.node_weights(), K).reshape(3, 3 * fib.n_nodes)
    return W / (8.0 * np.pi * mu)


def near_fiber_weights(fib, target, mu, include_doublet=False):
    """Panel-refined quadrature as a (3, 3n) map (fiber.py:514-565)."""
    target = np.asarray(target, dtype=float)
    _, _, d = nearest_centerline_point(fib, target)
    if d < fib.eps * fib.L:
        raise InsideFiberError("target overlaps the fiber surface")
    n = fib.n_nodes
    coeff = (fib.eps * fib.L) ** 2 / 2.0
    cx = [_coeffs(fib.X[:, c]) for c in range(3)]
    csa = _coeffs(fib.s_alpha)
    panels = [(-1.0, 1.0, 0)]
    al_all, w_all = [], []
    while panels:
        a, b, depth = panels.pop()
        probes = np.array([a, 0.5 * (a + b), b])
        px = np.stack([C.chebval(probes, c) for c in cx], axis=1)
        dmin = math.sqrt(((px - target) ** 2).sum(axis=1).min())
        if 0.5 * (b - a) * fib.L > dmin and depth < 14:
            mid = 0.5 * (a + b)
            panels.append((a, mid, depth + 1))
            panels.append((mid, b, depth + 1))
            continue
        al_all.append(0.5 * (a + b) + 0.5 * (b - a) * _GL10_X)
        w_all.append(0.5 * (b - a) * _GL10_W)
    al = np.concatenate(al_all)
    w = np.concatenate(w_all)
    Xp = np.stack([C.chebval(al, c) for c in cx], axis=1)
    sa = C.chebval(al, csa)
    P = _bary_rows(al, fib.p)
    K = _kernel_blocks(target[None, :] - Xp, include_doublet, coeff)
    W = np.einsum("g,gab,gj->ajb", w * sa, K, P).reshape(3, 3 * n) / (8.0 * np.pi * mu)
    shell = NEAR_SHELL_FACTOR * fib.L / fib.p
    x = (d - 0.8 * shell) / (0.2 * shell)
    if x > 0.0:
        xm = min(x, 1.0)
        wb = xm * xm * (3.0 - 2.0 * xm)
        W = (1.0 - wb) * W + wb * plain_fiber_weights(fib, target, mu, include_doublet)
    return W


def find_fiber_pairs(fibers, targets, target_groups, mu, include_doublet=True):
    """Near list [(t, l, Wnear - Wplain)] in the reference's order
    (system.py:564-586): fibers in order, targets ascending.  Candidate
    targets come from a k-d tree (exactly the min-node-distance < shell rule)."""
    from scipy.spatial import cKDTree

    out = []
    if not fibers or targets.shape[0] == 0:
        return out
    tree = cKDTree(targets)
    for l, fib in enumerate(fibers):
        shell = NEAR_SHELL_FACTOR * fib.L / fib.p
        hits = tree.query_ball_point(fib.X, r=shell)
        cand = np.unique(np.concatenate([np.asarray(h, dtype=np.int64) for h in hits]))
        if cand.size == 0:
            continue
        cand = cand[target_groups[cand] != l]
        if cand.size == 0:
            continue
        dd = targets[cand, None, :] - fib.X[None, :, :]
        d2 = (dd * dd).sum(axis=2).min(axis=1)
        for t in cand[d2 < shell * shell]:
            Wn = near_fiber_weights(fib, targets[t], mu, include_doublet=include_doublet)
            Wp = plain_fiber_weights(fib, targets[t], mu, include_doublet=include_doublet)
            out.append((int(t), l, Wn - Wp))
    return out
