"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference publishes no datasets; every configuration is synthetic.  The
laws follow BASELINE.json and SURVEY.md §8(d):

* straight fibers as in fiber.straight_fiber (fiber.py:225-232): minus end at
  `start`, X = start + s d with s = (alpha + 1) L / 2;
* directions: normalised standard normals; ball centres R u^(1/3) dir, cube
  centres uniform (the cloud_init law, system.py:458-467);
* optional centreline perturbation X(alpha) += sum_k c_k T_k(alpha),
  c_k ~ N(0, sigma^2) per component (reading "~N(0,1e-2)" as sigma = 1e-2);
* REJECTION SAMPLING: the reference raises OverlapError for targets within
  eps L of another fiber (fiber.py:526-528), so uniform draws fail
  (SURVEY.md fact 6).  A draw is rejected when it comes closer than `clear`
  to an accepted fiber: segment-segment distance for straight fibers
  ("segment"), node-node distance otherwise ("node").  clear = 2 eps L keeps
  near pairs ("near" variant, near-field maps exercised); clear = 1.05 * 1.5
  L/p empties the near list ("clean" variant: every node is outside every
  other fiber's near shell, system.py:564-577).
"""

import math
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
            X = X + V @ rng.normal(0.0, perturb, size=(n, 3))
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


def _node_sampling(rng, n_fibers, p, length, region, size, clear, perturb, max_draws):
    """Batched rejection on node-node distance: draw all fibers, find
    conflicting pairs with a k-d tree, keep the lower index of each conflict,
    redraw the rest, repeat."""
    from scipy.spatial import cKDTree

    n = p + 1
    V = C.chebvander(cheb_nodes(p), p) if perturb > 0 else None
    X = _draw(rng, n_fibers, p, length, region, size, perturb, V)
    draws = n_fibers
    pending = np.arange(n_fibers)
    while True:
        tree = cKDTree(X.reshape(-1, 3))
        pairs = tree.query_pairs(clear, output_type="ndarray")
        fa, fb = pairs[:, 0] // n, pairs[:, 1] // n
        keep = fa != fb
        fa, fb = np.minimum(fa[keep], fb[keep]), np.maximum(fa[keep], fb[keep])
        if fa.size == 0:
            break
        # greedy in index order: a fiber is rejected if it conflicts with a
        # lower-index fiber that itself survives
        order = np.lexsort((fa, fb))
        rejected = np.zeros(n_fibers, dtype=bool)
        pending_set = np.zeros(n_fibers, dtype=bool)
        pending_set[pending] = True
        for a, b in zip(fa[order], fb[order]):
            if rejected[a]:
                continue
            # only redraw fibers drawn in this round; earlier survivors stay
            if pending_set[b]:
                rejected[b] = True
            elif pending_set[a]:
                rejected[a] = True
        redo = np.nonzero(rejected)[0]
        if redo.size == 0:
            # conflicts among earlier survivors cannot happen; guard anyway
            redo = np.unique(fb)
        draws += redo.size
        if draws > max_draws:
            raise RuntimeError("rejection sampling did not converge; domain too dense")
        X[redo] = _draw(rng, redo.size, p, length, region, size, perturb, V)
        pending = redo
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
