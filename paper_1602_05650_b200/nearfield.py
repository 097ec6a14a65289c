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


# --------------------------------------------------------------- surfaces ----
# Nearly singular double-layer evaluation near a surface (body.py:371-519):
# a one-sided on-surface anchor (subtracted principal value plus the interior
# jump) and three off-surface samples at 1.5h, 2.25h, 3.375h on a six-fold
# refined mesh, combined by Lagrange interpolation along the normal ray and
# mapped back to the coarse nodal density by patchwise tensor interpolation.

from .body import GL01_NODES, make_surface  # noqa: E402

_REFINED = {}


def _lagrange(x, nodes):
    x = np.atleast_1d(np.asarray(x, dtype=float))
    c = np.ones((x.size, len(nodes)))
    for i in range(len(nodes)):
        for j in range(len(nodes)):
            if i != j:
                c[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return c


def refined(mesh, factor):
    key = (id(mesh), factor)
    if key not in _REFINED:
        nt, nph = mesh.patch_grid
        _REFINED[key] = (mesh, make_surface(mesh.shape, (nt * factor, nph * factor),
                                            center=mesh.center))
    return _REFINED[key][1]


def surface_point(mesh, theta, phi):
    R = mesh.shape[2](theta)
    return mesh.center + R * np.array([math.sin(theta) * math.cos(phi),
                                       math.sin(theta) * math.sin(phi), math.cos(theta)])


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

def device_fiber_pairs(geo, eps, targets, target_groups, mu, include_doublet=True):
    """Fiber near maps built on the device (sf_near_search + sf_near_fiber_weights).

    geo: system.FiberGeometry (device centrelines, s_alpha, L, weights);
    eps (nf,) device tensor; targets (nt,3) / target_groups (nt,) device.
    Returns (t, l, W): numpy pair indices in the reference's order (fibers in
    order, targets ascending, system.py:566-586) and the device tensor W
    (npairs, 3, 3n) of Wnear - Wplain.  Raises InsideFiberError like
    near_fiber_weights when a target overlaps a fiber.
    """
    import ctypes

    import torch

    from . import _native

    def ptr(t):
        return t.data_ptr() if t is not None and t.numel() else None

    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    dev = geo.X.device
    nf, n = geo.nf, geo.n
    nt = targets.shape[0]
    if nf == 0 or nt == 0:
        return (np.zeros(0, np.int64), np.zeros(0, np.int64),
                torch.zeros((0, 3, 3 * n), dtype=torch.float64, device=dev))
    p = n - 1
    center = geo.X.mean(dim=1).contiguous()
    shell = (NEAR_SHELL_FACTOR * geo.L / p).contiguous()
    bound = ((geo.X - center[:, None, :]).norm(dim=2).amax(dim=1) + shell).contiguous()
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    cap = max(1024, nt // 8)
    while True:
        pairs = torch.empty((cap, 2), dtype=torch.int64, device=dev)
        _native.call("sf_near_search", ptr(targets), ptr(target_groups), nt, ptr(geo.X), nf, n,
                     ptr(center), ptr(bound), ptr(shell), cap, ptr(pairs), ptr(count), st)
        found = int(count.item())
        if found <= cap:
            break
        cap = found + 1024
    pl_np, pt_np = (pairs[:found].cpu().numpy().T if found else (np.zeros(0, np.int64),) * 2)
    order = np.lexsort((pt_np, pl_np))
    pl_np, pt_np = pl_np[order], pt_np[order]
    W = device_fiber_weights(geo, eps, targets, pt_np, pl_np, mu, include_doublet)
    return pt_np.astype(np.int64), pl_np.astype(np.int64), W


def device_fiber_weights(geo, eps, targets, pt_np, pl_np, mu, include_doublet=True):
    """W_near - W_plain (3, 3n) for explicit (target, fiber) pairs
    (sf_near_fiber_weights; fiber.py:453-575), device tensor (k, 3, 3n)."""
    import ctypes

    import torch

    from . import _native, spectral

    def ptr(t):
        return t.data_ptr() if t is not None and t.numel() else None

    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    dev = geo.X.device
    n, p = geo.n, geo.n - 1
    k = len(pt_np)
    W = torch.empty((k, 3, 3 * n), dtype=torch.float64, device=dev)
    if k:
        nodes, _, _, _ = spectral.grid(p)
        glx, glw = np.polynomial.legendre.leggauss(10)
        consts = dict(Cmat=torch.tensor(spectral.coeff_matrix(p), dtype=torch.float64, device=dev),
                      nodes=torch.tensor(nodes, dtype=torch.float64, device=dev),
                      gl=torch.tensor(np.concatenate([glx, glw]), dtype=torch.float64, device=dev))
        pt = torch.as_tensor(np.asarray(pt_np, dtype=np.int64), device=dev)
        pl = torch.as_tensor(np.asarray(pl_np, dtype=np.int64), device=dev)
        info = torch.empty(k, dtype=torch.int32, device=dev)
        _native.call("sf_near_fiber_weights", ptr(pt), ptr(pl), k, ptr(targets), ptr(geo.X),
                     ptr(geo.s_alpha), ptr(geo.wcc), ptr(consts["Cmat"]), ptr(consts["nodes"]),
                     ptr(consts["gl"]), ptr(eps), ptr(geo.L), n, float(mu), int(include_doublet),
                     ptr(W), ptr(info), st)
        bad = info.cpu().numpy()
        if np.any(bad == 1):
            raise InsideFiberError("target overlaps the fiber surface")
        if np.any(bad == 2):
            raise RuntimeError("near-field panel refinement overflowed its buffer")
    return W


_DEV_MESH = {}          # (id(mesh), factor, device) -> (mesh, tensors); small LRU


def _device_mesh(mesh, factor, device):
    """Device arrays of the coarse mesh, its factor-x refinement and the
    fine-from-coarse interpolation coefficients (_interpolation_matrix)."""
    import torch
    key = (id(mesh), factor, str(device))
    hit = _DEV_MESH.pop(key, None)
    if hit is not None:
        _DEV_MESH[key] = hit
        return hit[1]
    f64 = dict(dtype=torch.float64, device=device)
    nt, nph = mesh.patch_grid
    if factor == 1:
        fine = mesh
        coef = np.zeros((mesh.n_nodes, 8))
        q = np.arange(mesh.n_nodes) % 16
        coef[np.arange(mesh.n_nodes), q // 4] = 1.0
        coef[np.arange(mesh.n_nodes), 4 + q % 4] = 1.0
    else:
        fine = refined(mesh, factor)
        theta = np.asarray(fine.thetas, dtype=float)
        phi = np.asarray(fine.phis, dtype=float) % (2.0 * np.pi)
        dth, dph = np.pi / nt, 2.0 * np.pi / nph
        it = np.minimum((theta / dth).astype(int), nt - 1)
        ip = np.minimum((phi / dph).astype(int), nph - 1)
        fpatch = np.arange(fine.n_nodes) // 16
        if not (np.array_equal(it, (fpatch // (nph * factor)) // factor)
                and np.array_equal(ip, (fpatch % (nph * factor)) // factor)):
            raise RuntimeError("refined patches do not nest in the coarse patches")
        coef = np.concatenate([_lagrange((theta - it * dth) / dth, GL01_NODES),
                               _lagrange((phi - ip * dph) / dph, GL01_NODES)], axis=1)
    t = dict(cnodes=torch.as_tensor(mesh.nodes, **f64).contiguous(),
             cnrm=torch.as_tensor(mesh.normals, **f64).contiguous(),
             cw=torch.as_tensor(mesh.weights, **f64).contiguous(),
             fnodes=torch.as_tensor(fine.nodes, **f64).contiguous(),
             fnrm=torch.as_tensor(fine.normals, **f64).contiguous(),
             fw=torch.as_tensor(fine.weights, **f64).contiguous(),
             fcoef=torch.as_tensor(np.ascontiguousarray(coef), **f64))
    _DEV_MESH[key] = (mesh, t)
    while len(_DEV_MESH) > 8:
        _DEV_MESH.pop(next(iter(_DEV_MESH)))
    return t


def device_surface_weights(mesh, targets, mu, device, interior_jump=True, upsample=6):
    """near_surface_weights - plain_surface_weights (body.py:479-519) for the
    given targets of one mesh, built on the device (sf_near_surface_weights).
    The nearest surface point (a scalar golden-section search on the
    profile R(theta), body.py:371-423) and the per-target Lagrange scalars
    are host work; every O(N_fine) sum runs on the B200.  Returns a device
    tensor (k, 3, 3N)."""
    import ctypes

    import torch

    from . import _native

    def ptr(x):
        return x.data_ptr() if x is not None and x.numel() else None
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f64 = dict(dtype=torch.float64, device=device)
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    k_all = targets.shape[0]
    W_all = torch.empty((k_all, 3, 3 * mesh.n_nodes), **f64)
    groups = {1: [], upsample: []}
    per_pair = []
    nt_, nph_ = mesh.patch_grid
    for j, tgt in enumerate(targets):
        th0, ph0, x0, sd = nearest_surface_point(mesh, tgt)
        dist = abs(sd)
        if dist < 1e-8 * mesh.h:                      # on the surface: coarse map
            fct, jump = 1, ((1.0 / mu) if interior_jump else 0.0)
            ell = np.array([1.0, 0.0, 0.0, 0.0])
            pts = np.zeros((3, 3))
        else:
            fct = upsample
            jump = (1.0 / mu) if (sd < 0 and interior_jump) else 0.0
            ndir = (tgt - x0) / dist
            c = 1.5 * mesh.h
            dists = np.array([0.0, c, 1.5 * c, 2.25 * c])
            ell = _lagrange(dist, dists)[0]
            pts = x0[None, :] + dists[1:, None] * ndir[None, :]
        gt, gp = nt_ * fct, nph_ * fct
        dth, dph = np.pi / gt, 2.0 * np.pi / gp
        phw = ph0 % (2.0 * np.pi)
        it = min(int(th0 / dth), gt - 1)
        ip = min(int(phw / dph), gp - 1)
        cu = _lagrange((th0 - it * dth) / dth, GL01_NODES)[0]
        cv = _lagrange((phw - ip * dph) / dph, GL01_NODES)[0]
        groups[fct].append(j)
        per_pair.append((tgt, x0, pts, ell, jump, it * gp + ip, np.outer(cu, cv).ravel()))
    for fct, js in groups.items():
        if not js:
            continue
        m = _device_mesh(mesh, fct, device)
        k = len(js)
        cols = list(zip(*[per_pair[j] for j in js]))
        trg = torch.as_tensor(np.stack(cols[0]), **f64)
        x0 = torch.as_tensor(np.stack(cols[1]), **f64)
        pts = torch.as_tensor(np.stack(cols[2]), **f64)
        ell = torch.as_tensor(np.stack(cols[3]), **f64)
        jump = torch.as_tensor(np.array(cols[4], dtype=float), **f64)
        r0p = torch.as_tensor(np.array(cols[5], dtype=np.int64), device=device)
        r0c = torch.as_tensor(np.stack(cols[6]), **f64)
        work = torch.empty(k * (9 + 148 * 9), **f64)
        W = torch.empty((k, 3, 3 * mesh.n_nodes), **f64)
        _native.call("sf_near_surface_weights", ptr(m["cnodes"]), ptr(m["cnrm"]), ptr(m["cw"]),
                     nt_, nph_, ptr(m["fnodes"]), ptr(m["fnrm"]), ptr(m["fw"]), ptr(m["fcoef"]),
                     fct, k, ptr(trg), ptr(x0), ptr(pts), ptr(ell), ptr(jump), ptr(r0p), ptr(r0c),
                     float(mu), ptr(work), ptr(W), st)
        W_all[torch.as_tensor(js, device=device)] = W
    return W_all


def device_surface_pairs(surfaces, trg, tgrp, mu, device, upsample=6, surface_arrays=None):
    """find_surface_pairs with the search and the maps on the device
    (device_surface_weights).  trg (nt, 3) and tgrp (nt,) are device
    tensors.  Candidates: other constituents' targets in the radial band of
    the mesh, then the nearest node closer than 1.5 h (system.py:588-613),
    both on the device; only the near targets' coordinates come back to the
    host for the per-target nearest-point preparation.  Returns
    [(t, si, W)] in the reference's order with W (3, 3N) device rows."""
    import torch
    f64 = dict(dtype=torch.float64, device=device)
    out = []
    for si, (mesh, group, is_periphery) in enumerate(surfaces):
        if surface_arrays is not None:
            nodes = surface_arrays[si][0]
        else:
            nodes = torch.as_tensor(mesh.nodes, **f64)
        center = getattr(mesh, "center_dev", None)
        if center is None:
            center = torch.as_tensor(mesh.center, **f64)
        shell = 1.5 * mesh.h
        rel = torch.linalg.vector_norm(trg - center, dim=1)
        rho_nodes = torch.linalg.vector_norm(nodes - center, dim=1)
        band = (tgrp != group) & (rel >= rho_nodes.min() - shell) & (rel <= rho_nodes.max() + shell)
        cand = torch.nonzero(band).reshape(-1)
        if cand.numel() == 0:
            continue
        d2 = torch.empty(cand.numel(), **f64)
        for a in range(0, cand.numel(), 128):          # nearest node, brute force in chunks
            c = trg[cand[a:a + 128]]
            d2[a:a + 128] = ((c[:, None, :] - nodes[None, :, :]) ** 2).sum(dim=2).min(dim=1).values
        near = cand[d2 < shell * shell].cpu().numpy()
        if near.size == 0:
            continue
        W = device_surface_weights(mesh, trg[torch.as_tensor(near, device=device)].cpu().numpy(),
                                   mu, device, interior_jump=is_periphery, upsample=upsample)
        out.extend((int(t), si, W[j]) for j, t in enumerate(near))
    return out
