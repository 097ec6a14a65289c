"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference publishes no datasets; every configuration is synthetic.  The
laws follow BASELINE.json and SURVEY.md §8(d):

* straight fibers as in fiber.straight_fiber (fiber.py:225-232): minus end at
  `start`, X = start + s d with s = (alpha + 1) L / 2;
* directions: normalised standard normals; ball centres R u^(1/3) dir, cube
  centres uniform (the cloud_init law, system.py:458-467);
* optional centreline perturbation X(alpha) += sum_k c_k T_k(alpha),
  c_k ~ N(0, sigma^2) per component with sigma = 1e-2 (our reading of
  "~N(0,1e-2)") on the lowest PERTURB_MODES = 4 Chebyshev modes.  Drawing all
  p+1 coefficients with that variance makes the centreline a zig-zag at the
  node scale (arclength 8-12 for a length-1 fiber at p = 63, measured), i.e.
  not a resolved fiber of length 1; the low-mode reading keeps L = 1 +- O(1e-2);
* REJECTION SAMPLING: the reference raises OverlapError for targets within
  eps L of another fiber (fiber.py:526-528), so uniform draws fail
  (SURVEY.md fact 6).  A draw is rejected when it comes closer than `clear`
  to an accepted fiber: segment-segment distance for straight fibers
  ("segment"), node-node distance otherwise ("node").  clear = 2 eps L keeps
  near pairs ("near" variant, near-field maps exercised); clear = 1.05 * 1.5
  L/p empties the near list ("clean" variant: every node is outside every
  other fiber's near shell, system.py:564-577).
"""

from dataclasses import dataclass, field

import numpy as np
from numpy.polynomial import chebyshev as C

from .spectral import cheb_nodes


@dataclass
class FiberCloud:
    X: np.ndarray            # (nf, n, 3)
    p: int
    eps: float
    E: float
    length: float
    seed: int
    draws: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n_fibers(self):
        return self.X.shape[0]

    @property
    def n_nodes(self):
        return self.X.shape[1]

    @property
    def n_points(self):
        return self.X.shape[0] * self.X.shape[1]


def straight_centerline(p, start, direction, length):
    d = np.asarray(direction, dtype=float)
    d = d / np.linalg.norm(d)
    s = (cheb_nodes(p) + 1.0) * (length / 2.0)
    return np.asarray(start, dtype=float)[None, :] + s[:, None] * d[None, :]


def _seg_dist(p0, p1, q0, q1):
    """Min distance between segment p0p1 and each segment q0[k]q1[k]."""
    d1 = p1 - p0
    d2 = q1 - q0
    r = p0[None, :] - q0
    a = d1 @ d1
    e = (d2 * d2).sum(axis=1)
    f = (d2 * r).sum(axis=1)
    c = r @ d1
    b = d2 @ d1
    denom = a * e - b * b
    s = np.where(denom > 1e-300, np.clip((b * f - c * e) / np.where(denom > 1e-300, denom, 1.0), 0, 1), 0.0)
    t = (b * s + f) / np.where(e > 0, e, 1.0)
    t_c = np.clip(t, 0, 1)
    s = np.where(t < 0, np.clip(-c / a, 0, 1), np.where(t > 1, np.clip((b - c) / a, 0, 1), s))
    t = t_c
    cp = p0[None, :] + s[:, None] * d1[None, :]
    cq = q0 + t[:, None] * d2
    return np.sqrt(((cp - cq) ** 2).sum(axis=1))


PERTURB_MODES = 4


def _draw(rng, k, p, length, region, size, perturb, V):
    """k candidate centrelines (k, n, 3) from the placement laws."""
    n = p + 1
    out = np.empty((k, n, 3))
    for i in range(k):
        if region == "ball":
            cdir = rng.standard_normal(3)
            cdir /= np.linalg.norm(cdir)
            centre = size * rng.random() ** (1.0 / 3.0) * cdir
        else:
            centre = rng.uniform(-size, size, 3)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        X = straight_centerline(p, centre - 0.5 * length * d, d, length)
        if perturb > 0:
            coef = np.zeros((n, 3))
            coef[:PERTURB_MODES] = rng.normal(0.0, perturb, size=(PERTURB_MODES, 3))
            X = X + V @ coef
        out[i] = X
    return out


def _segment_sampling(rng, n_fibers, p, length, region, size, clear, max_draws):
    """Sequential rejection on exact segment-segment distance (straight fibers)."""
    cell = length + clear
    grid = {}
    Xs, segs = [], []
    draws = 0
    while len(Xs) < n_fibers:
        draws += 1
        if draws > max_draws:
            raise RuntimeError("rejection sampling did not converge; domain too dense")
        X = _draw(rng, 1, p, length, region, size, 0.0, None)[0]
        centre = 0.5 * (X[0] + X[-1])
        key = tuple(np.floor(centre / cell).astype(int))
        neigh = []
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dz in (-1, 0, 1):
                    neigh.extend(grid.get((key[0] + dx, key[1] + dy, key[2] + dz), ()))
        if neigh:
            q = np.asarray([segs[k] for k in neigh])
            if _seg_dist(X[-1], X[0], q[:, 0], q[:, 1]).min() < clear:
                continue
        grid.setdefault(key, []).append(len(Xs))
        Xs.append(X)
        segs.append((X[-1], X[0]))
    return np.stack(Xs), draws


def _node_sampling(rng, n_fibers, p, length, region, size, clear, perturb, max_draws,
                   upsample=4):
    """Batched rejection on centreline-sample distance: draw all fibers,
    resample each centreline at `upsample` x the Chebyshev nodes (the nodes
    included), find conflicting pairs with a k-d tree, keep the lower index of
    each conflict, redraw the rest, repeat.  Sampling the centreline (not only
    the nodes) keeps every node outside other fibers' radius as well."""
    from scipy.spatial import cKDTree

    n = p + 1
    V = C.chebvander(cheb_nodes(p), p) if perturb > 0 else None
    # nodal values -> values at the refined extremal points (nodes are a subset)
    fine = np.cos(np.pi * np.arange(upsample * p + 1) / (upsample * p))
    E = C.chebvander(fine, p) @ np.linalg.inv(C.chebvander(cheb_nodes(p), p))
    nfine = fine.size
    def refine(Xs):
        m = Xs.shape[0]
        return (E @ Xs.transpose(1, 0, 2).reshape(n, -1)).reshape(nfine, m, 3).transpose(1, 0, 2)

    X = _draw(rng, n_fibers, p, length, region, size, perturb, V)
    F = refine(X)
    draws = n_fibers
    # round 0: all pairs among the initial draws; keep the lower index
    tree = cKDTree(F.reshape(-1, 3))
    pairs = tree.query_pairs(clear, output_type="ndarray")
    fa, fb = pairs[:, 0] // nfine, pairs[:, 1] // nfine
    keep = fa != fb
    fa, fb = np.minimum(fa[keep], fb[keep]), np.maximum(fa[keep], fb[keep])
    rejected = np.zeros(n_fibers, dtype=bool)
    for a, b in sorted(set(zip(fa.tolist(), fb.tolist())), key=lambda ab: (ab[1], ab[0])):
        if not rejected[a]:
            rejected[b] = True
    redo = np.nonzero(rejected)[0]
    # later rounds: redraw the rejected fibers and test them against the fixed
    # survivors (old tree, stale entries of redrawn fibers ignored) and each other
    while redo.size:
        draws += redo.size
        if draws > max_draws:
            raise RuntimeError("rejection sampling did not converge; domain too dense")
        X[redo] = _draw(rng, redo.size, p, length, region, size, perturb, V)
        F[redo] = refine(X[redo])
        in_redo = np.zeros(n_fibers, dtype=bool)
        in_redo[redo] = True
        bad = np.zeros(n_fibers, dtype=bool)
        hits = tree.query_ball_point(F[redo].reshape(-1, 3), r=clear)
        for k, h in enumerate(hits):
            if h:
                ids = np.asarray(h) // nfine
                if np.any(~in_redo[ids]):
                    bad[redo[k // nfine]] = True
        small = cKDTree(F[redo].reshape(-1, 3))
        pr = small.query_pairs(clear, output_type="ndarray")
        ra, rb = redo[pr[:, 0] // nfine], redo[pr[:, 1] // nfine]
        keep = ra != rb
        for a, b in sorted(set(zip(np.minimum(ra[keep], rb[keep]).tolist(),
                                   np.maximum(ra[keep], rb[keep]).tolist())),
                           key=lambda ab: (ab[1], ab[0])):
            if not bad[a]:
                bad[b] = True
        accepted = redo[~bad[redo]]
        if accepted.size:
            tree = cKDTree(F.reshape(-1, 3)) if accepted.size > 0 else tree
        redo = redo[bad[redo]]
    return X, draws


def fiber_cloud(n_fibers, p, length=1.0, eps=1e-2, E=1.0, region="cube", size=2.0, seed=0,
                clear=None, check="segment", perturb=0.0, max_draws_factor=1000):
    """Rejection-sampled cloud of fibers; returns a FiberCloud."""
    rng = np.random.default_rng(seed)
    if clear is None:
        clear = 2.0 * eps * length
    max_draws = max_draws_factor * n_fibers
    if check == "segment":
        if perturb > 0:
            raise ValueError("segment rejection needs straight fibers")
        X, draws = _segment_sampling(rng, n_fibers, p, length, region, size, clear, max_draws)
    else:
        X, draws = _node_sampling(rng, n_fibers, p, length, region, size, clear, perturb,
                                  max_draws)
    return FiberCloud(X, p, eps, E, length, seed, draws,
                      dict(region=region, size=size, clear=clear, check=check, perturb=perturb))


def clean_clear(p, length=1.0):
    return 1.05 * 1.5 * length / p


# name -> keyword arguments of fiber_cloud (BASELINE.json configs)
CONFIGS = {
    # C1: 64 fibers, L=1, eps=1e-2, 32 points, centres in [-2,2]^3
    "c1": dict(n_fibers=64, p=31, eps=1e-2, E=1.0, region="cube", size=2.0),
    "c1_clean": dict(n_fibers=64, p=31, eps=1e-2, E=1.0, region="cube", size=2.0,
                     clear=clean_clear(31), check="node"),
    # C3: 4096 fibers x 64 points, eps=5e-3, E=1e-2, ball R=10, perturbed centrelines
    "c3": dict(n_fibers=4096, p=63, eps=5e-3, E=1e-2, region="ball", size=10.0,
               perturb=1e-2, clear=clean_clear(63), check="node"),
    "c3_scaled": dict(n_fibers=512, p=63, eps=5e-3, E=1e-2, region="ball", size=5.0,
                      perturb=1e-2, clear=clean_clear(63), check="node"),
    # C5: 16384 fibers x 64 points = 1,048,576 points, ball R=20
    "c5": dict(n_fibers=16384, p=63, eps=5e-3, E=1e-2, region="ball", size=20.0,
               perturb=1e-2, clear=clean_clear(63), check="node"),
}


def make(name, seed=0, **overrides):
    kw = dict(CONFIGS[name])
    kw.update(overrides)
    return fiber_cloud(seed=seed, **kw)


def forces(cloud, seed=1):
    """i.i.d. N(0,1) force densities per point (BASELINE.json C1)."""
    return np.random.default_rng(seed).standard_normal(cloud.X.shape)


def aster_layout(n_fibers=1024, radius=0.5, standoff=1.3, center=(0.0, 0.0, 0.0),
                 min_sep=0.05, seed=0, layout="random"):
    """Attachment points (n_fibers, 3) and unit directions (n_fibers, 3) of a
    radial aster (BASELINE config 2, config 4's centrosome).

    layout "random": uniform directions (normalised Gaussians) with rejection
    of attachment points closer than `min_sep` (uniform draws overlap,
    SURVEY.md fact 6); "fibonacci": a Fibonacci spiral over the sphere (the
    law of the reference's aster_attachment_layout, system.py:428-443).
    Attachment at standoff * radius (the reference default 1.3)."""
    center = np.asarray(center, dtype=float)
    rng = np.random.default_rng(seed)
    r_att = standoff * radius
    if layout == "fibonacci":
        k = np.arange(n_fibers)
        z = 1.0 - 2.0 * (k + 0.5) / n_fibers
        rho = np.sqrt(1.0 - z * z)
        phi = k * (np.pi * (3.0 - np.sqrt(5.0)))
        dirs = np.stack([rho * np.cos(phi), rho * np.sin(phi), z], axis=1)
    else:
        dirs = []
        pts = []
        draws = 0
        while len(dirs) < n_fibers:
            draws += 1
            if draws > 1000 * n_fibers:
                raise RuntimeError("aster rejection sampling did not converge")
            d = rng.standard_normal(3)
            d /= np.linalg.norm(d)
            x = r_att * d
            if pts and np.min(np.linalg.norm(np.asarray(pts) - x, axis=1)) < min_sep:
                continue
            dirs.append(d)
            pts.append(x)
        dirs = np.asarray(dirs)
    return center[None, :] + r_att * dirs, dirs


def aster(n_fibers=1024, p=31, radius=0.5, standoff=1.3, center=(0.0, 0.0, 0.0), eps=1e-2,
          E=1.0, length=1.0, mesh_res=(8, 8), min_sep=0.05, motor_force=1.0, seed=0,
          layout="random"):
    """BASELINE config 2 (and 4's centrosome): fibers clamped radially to a
    rigid sphere (attachment from aster_layout), plus-end force of magnitude
    `motor_force` along the initial tangent (a fixed vector, as
    PrescribedForceTorque stores it, fiber.py:58-63).  Returns a SystemState
    of this package."""
    from . import body
    from .fiber import ClampedToBody, PrescribedForceTorque, straight_fiber
    from .system import SystemState

    part = body.RigidParticle(body.make_surface(body.sphere_shape(radius), mesh_res,
                                                center=tuple(float(c) for c in center)))
    pts, dirs = aster_layout(n_fibers, radius, standoff, center, min_sep, seed, layout)
    fibs = []
    for x0, d in zip(pts, dirs):
        fibs.append(straight_fiber(p, x0, d, length, eps=eps, E=E,
                                   bc_minus=ClampedToBody(0, x0, d),
                                   bc_plus=PrescribedForceTorque(motor_force * d)))
    return SystemState(fibs, [part])


def cloud_state(name="c3_scaled", seed=0, f0=1.0, direction=(0.0, 0.0, -1.0), **overrides):
    """Sedimenting cloud (BASELINE configs 3/5): free fibers under a uniform
    force density (0,0,-1) (UniformBodyForce, system.py:40-54)."""
    from .fiber import Fiber
    from .system import SystemState, UniformBodyForce

    cl = make(name, seed=seed, **overrides)
    fibs = [Fiber(X, eps=cl.eps, E=cl.E) for X in cl.X]
    return SystemState(fibs, force_models=[UniformBodyForce(f0, direction)])


def confined_aster(n_fibers=2048, p=31, centrosome_radius=0.3, centrosome_center=(0.5, 0.0, 0.0),
                   centrosome_res=(8, 8), periphery_radius=2.0, periphery_res=(40, 64),
                   standoff=1.3, eps=1e-2, E=1.0, motor_force=1.0, periphery_mesh="patch"):
    """BASELINE config 4: fibers clamped radially (reference Fibonacci layout,
    system.py:428-443) to a centrosome sphere inside a confining sphere.  The
    icosphere of the baseline is not expressible in the reference; the
    (40,64)-patch sphere has 40,960 nodes and is the default.
    periphery_mesh="ico" uses the literal 40,962-vertex icosphere instead
    (body.make_icosphere, 6 subdivisions; beyond the reference)."""
    from . import body
    st = aster(n_fibers=n_fibers, p=p, radius=centrosome_radius, standoff=standoff,
               center=centrosome_center, eps=eps, E=E, mesh_res=centrosome_res,
               motor_force=motor_force, layout="fibonacci")
    if periphery_mesh == "ico":
        per = body.Periphery(body.make_icosphere(periphery_radius, 6))
    else:
        per = body.Periphery(body.make_surface(body.sphere_shape(periphery_radius),
                                               periphery_res))
    from .system import SystemState
    return SystemState(st.fibers, st.particles, per)
