"""Near-field correction maps, built on the device.

Targets closer than 1.5 L/p to another fiber, or 1.5 h to a surface, get a
small linear map W that replaces the plain collocation sum (the reference's
algorithm: fiber.py:453-575, body.py:371-519, system.py:564-613).  Fiber
maps: candidate search, nearest centreline point, adaptive Gauss-Legendre
panels, barycentric resampling and the smoothstep blend all run in
sf_near_search / sf_near_fiber_weights.  Surface maps: the radial-band and
nearest-node search run on the device (device_surface_pairs); per near
target the nearest point on the profile R(theta) comes from the reference's
own scalar search (slenderflow.body.nearest_surface_point, via
_reference.py), and every O(N_fine) sum -- fine-mesh stresslet sums, row
sums, extrapolation, fine-to-coarse contraction -- runs in
sf_near_surface_weights.  The maps are applied every matvec by sf_near_apply.
(The host restatement of these maps is test infrastructure:
oracle/nearfield.py.)
"""

import math

import numpy as np

from . import spectral
from .body import GL01_NODES, make_surface
from .fiber import InsideFiberError

NEAR_SHELL_FACTOR = 1.5


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

    from . import _native, _reference

    def ptr(x):
        return x.data_ptr() if x is not None and x.numel() else None
    if getattr(mesh, "patch_grid", None) is None:
        from .body import GeometryError
        raise GeometryError("a target lies in the near shell of a surface without patches "
                            "(icosphere); near-surface maps need a make_surface mesh")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    f64 = dict(dtype=torch.float64, device=device)
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    k_all = targets.shape[0]
    W_all = torch.empty((k_all, 3, 3 * mesh.n_nodes), **f64)
    groups = {1: [], upsample: []}
    per_pair = []
    nt_, nph_ = mesh.patch_grid
    nearest_surface_point = _reference.module("body").nearest_surface_point
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
