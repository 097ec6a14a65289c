"""ORACLE (test infrastructure only): host restatement of the reference's
near-field correction maps (fiber.py:453-575, body.py:371-519,
system.py:564-613), checked against golden maps made by the reference
itself (tests/golden/make_golden.py) and used as the checker of the device
construction (paper_1602_05650_b200.nearfield, sf_near_*).  Never imported
by the product.

Fiber maps: nearest centreline point by refined sampling plus golden-section
search, adaptive bisection into 10-point Gauss-Legendre panels until each is
shorter than its distance to the target, barycentric resampling of the nodal
density and a smoothstep blend back to the plain sum near the shell
boundary.  Surface maps: nearest point on R(theta), fine-mesh quadrature
with the interior jump, extrapolation along the normal.
"""

import math

import numpy as np
from numpy.polynomial import chebyshev as C

from paper_1602_05650_b200 import spectral
from paper_1602_05650_b200.body import GL01_NODES
from paper_1602_05650_b200.fiber import InsideFiberError
from paper_1602_05650_b200.nearfield import _lagrange, refined, surface_point

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


# --------------------------------------------------------------- surfaces ----
# Nearly singular double-layer evaluation near a surface (body.py:371-519):
# a one-sided on-surface anchor (subtracted principal value plus the interior
# jump) and three off-surface samples at 1.5h, 2.25h, 3.375h on a six-fold
# refined mesh, combined by Lagrange interpolation along the normal ray and
# mapped back to the coarse nodal density by patchwise tensor interpolation.


def nearest_surface_point(mesh, target):
    """(theta, phi, point, signed distance) (body.py:371-423)."""
    t = np.asarray(target, dtype=float)
    rel = t - mesh.center
    rho = math.hypot(rel[0], rel[1])
    phi = math.atan2(rel[1], rel[0]) if rho > 1e-14 else 0.0
    R = mesh.shape[2]

    def dist2(th):
        r = float(R(th))
        a = r * math.sin(th) - rho
        b = r * math.cos(th) - rel[2]
        return a * a + b * b

    scan = np.linspace(0.0, math.pi, 65)
    vals = [dist2(x) for x in scan]
    i0 = int(np.argmin(vals))
    lo, hi = scan[max(i0 - 1, 0)], scan[min(i0 + 1, 64)]
    for _ in range(40):
        m1 = lo + 0.382 * (hi - lo)
        m2 = lo + 0.618 * (hi - lo)
        if dist2(m1) < dist2(m2):
            hi = m2
        else:
            lo = m1
    th0 = 0.5 * (lo + hi)
    fd = 1e-6
    for _ in range(3):
        gr = (dist2(th0 + fd) - dist2(th0 - fd)) / (2 * fd)
        gpp = (dist2(th0 + fd) - 2 * dist2(th0) + dist2(th0 - fd)) / fd ** 2
        if gpp <= 0:
            break
        cand = min(max(th0 - gr / gpp, 0.0), math.pi)
        if dist2(cand) <= dist2(th0):
            th0 = cand
    x0 = surface_point(mesh, th0, phi)
    d = float(np.linalg.norm(t - x0))
    r_t = np.linalg.norm(rel)
    th_t = math.acos(min(max(rel[2] / r_t, -1.0), 1.0)) if r_t > 0 else 0.0
    inside = r_t < float(R(th_t))
    return th0, phi, x0, (-d if inside else d)


def plain_surface_weights(mesh, target, mu):
    """Stresslet quadrature at one target as a (3, 3N) map (body.py:437-448)."""
    r = np.asarray(target, dtype=float)[None, :] - mesh.nodes
    d2 = (r * r).sum(axis=1)
    live = d2 > 1e-24
    nr = (mesh.normals * r).sum(axis=1)
    scal = np.zeros(mesh.n_nodes)
    scal[live] = (-3.0 / (4.0 * np.pi * mu)) * mesh.weights[live] * nr[live] \
        / (d2[live] ** 2 * np.sqrt(d2[live]))
    W = scal[None, :, None] * r.T[:, :, None] * r[None, :, :]
    return W.reshape(3, 3 * mesh.n_nodes)


def _interp_row(mesh, theta, phi):
    nt, nph = mesh.patch_grid
    dth, dph = np.pi / nt, 2.0 * np.pi / nph
    phi = phi % (2.0 * np.pi)
    it = min(int(theta / dth), nt - 1)
    ip = min(int(phi / dph), nph - 1)
    cu = _lagrange((theta - it * dth) / dth, GL01_NODES)[0]
    cv = _lagrange((phi - ip * dph) / dph, GL01_NODES)[0]
    row = np.zeros(mesh.n_nodes)
    row[(it * nph + ip) * 16 + np.arange(16)] = np.outer(cu, cv).ravel()
    return row


def _subtracted_rows_at(mesh, theta, phi, mu, jump):
    x0 = surface_point(mesh, theta, phi)
    rows = plain_surface_weights(mesh, x0, mu).reshape(3, mesh.n_nodes, 3)
    RS = rows.sum(axis=1)
    r0 = _interp_row(mesh, theta, phi)
    rows -= RS[:, None, :] * r0[None, :, None]
    if jump != 0.0:
        rows += jump * np.eye(3)[:, None, :] * r0[None, :, None]
    return rows


def _interpolation_matrix(mesh, fine):
    from scipy import sparse
    theta = np.asarray(fine.thetas, dtype=float)
    phi = np.asarray(fine.phis, dtype=float) % (2.0 * np.pi)
    nt, nph = mesh.patch_grid
    dth, dph = np.pi / nt, 2.0 * np.pi / nph
    it = np.minimum((theta / dth).astype(int), nt - 1)
    ip = np.minimum((phi / dph).astype(int), nph - 1)
    cu = _lagrange((theta - it * dth) / dth, GL01_NODES)
    cv = _lagrange((phi - ip * dph) / dph, GL01_NODES)
    vals = np.einsum("mi,mj->mij", cu, cv).reshape(theta.size, 16)
    cols = ((it * nph + ip) * 16)[:, None] + np.arange(16)
    rows = np.repeat(np.arange(theta.size), 16)
    return sparse.csr_matrix((vals.ravel(), (rows, cols.ravel())),
                             shape=(theta.size, mesh.n_nodes))


_INTERP = {}


def near_surface_weights(mesh, target, mu, interior_jump=True, upsample=6):
    """(3, 3N) near-surface map (body.py:479-519)."""
    target = np.asarray(target, dtype=float)
    th0, ph0, x0, signed_d = nearest_surface_point(mesh, target)
    d = abs(signed_d)
    interior = signed_d < 0
    if d < 1e-8 * mesh.h:
        jump = (1.0 / mu) if interior_jump else 0.0
        return _subtracted_rows_at(mesh, th0, ph0, mu, jump).reshape(3, 3 * mesh.n_nodes)
    fine = refined(mesh, upsample) if upsample > 1 else mesh
    jump = (1.0 / mu) if (interior and interior_jump) else 0.0
    Wf = _subtracted_rows_at(fine, th0, ph0, mu, jump)
    normal_dir = (target - x0) / d
    c = 1.5 * mesh.h
    dists = np.array([0.0, c, 1.5 * c, 2.25 * c])
    ell = _lagrange(d, dists)[0]
    Wf = ell[0] * Wf
    for k in range(1, 4):
        pt = x0 + dists[k] * normal_dir
        Wf += ell[k] * plain_surface_weights(fine, pt, mu).reshape(3, fine.n_nodes, 3)
    if fine is mesh:
        return Wf.reshape(3, 3 * mesh.n_nodes)
    key = (id(mesh), id(fine))
    if key not in _INTERP:
        _INTERP[key] = (mesh, fine, _interpolation_matrix(mesh, fine))
    B = _INTERP[key][2]
    W = np.empty((3, mesh.n_nodes, 3))
    for a in range(3):
        for b in range(3):
            W[a, :, b] = B.T @ Wf[a, :, b]
    return W.reshape(3, 3 * mesh.n_nodes)


def find_surface_pairs(surfaces, targets, target_groups, mu):
    """Near-surface list [(t, si, Wnear - Wplain)] in the reference's order
    (system.py:588-613); surfaces: [(mesh, group, is_periphery)]."""
    out = []
    for si, (mesh, group, is_periphery) in enumerate(surfaces):
        others = target_groups != group
        shell = 1.5 * mesh.h
        rel = np.linalg.norm(targets - mesh.center, axis=1)
        rho_nodes = np.linalg.norm(mesh.nodes - mesh.center, axis=1)
        band = others & (rel >= rho_nodes.min() - shell) & (rel <= rho_nodes.max() + shell)
        cand = np.nonzero(band)[0]
        if cand.size == 0:
            continue
        from scipy.spatial import cKDTree
        d, _ = cKDTree(mesh.nodes).query(targets[cand], k=1)
        for t in cand[d * d < shell * shell]:
            Wn = near_surface_weights(mesh, targets[t], mu, interior_jump=is_periphery)
            Wp = plain_surface_weights(mesh, targets[t], mu)
            out.append((int(t), si, Wn - Wp))
    return out


# ------------------------------------------------------------------ device ----

