"""Chebyshev collocation constants per order p (host setup, computed once).

Conventions follow the reference (/root/reference/pkg/src/slenderflow/
spectral.py): extremal nodes cos(k pi / p) ordered +1 -> -1, node 0 is the
plus end (s = L), node p the minus end (s = 0).  The per-fiber, per-step work
(arclength, tangents, D_s powers, weights) runs on the device from these
constant matrices.
"""

import functools

import numpy as np
from numpy.polynomial import chebyshev as C
from scipy.fft import dct


class InvalidOrderError(ValueError):
    pass


class DegenerateFiberError(ValueError):
    pass


def cheb_nodes(p):
    """Extremal points, symmetrised to be exactly antisymmetric (spectral.py:24-34)."""
    if int(p) != p or p < 1:
        raise InvalidOrderError(f"order must be an integer >= 1, got {p}")
    p = int(p)
    a = np.cos(np.pi * np.arange(p + 1) / p)
    return 0.5 * (a - a[::-1])


def values_to_coeffs(v):
    """Chebyshev coefficients of the interpolant through nodal values (DCT-I)."""
    v = np.asarray(v, dtype=float)
    p = v.shape[0] - 1
    c = dct(v, type=1, axis=0) / p
    c[0] *= 0.5
    c[-1] *= 0.5
    return c


@functools.lru_cache(maxsize=None)
def grid(p):
    """(nodes, Clenshaw-Curtis weights, D_alpha, arclength-integration matrix)."""
    if int(p) != p or p < 4:
        raise InvalidOrderError(f"grid order must be an integer >= 4, got {p}")
    p = int(p)
    n = p + 1
    nodes = cheb_nodes(p)
    eye = np.eye(n)
    # coefficient map, one nodal unit vector at a time
    Cmat = np.stack([values_to_coeffs(eye[:, j]) for j in range(n)], axis=1)
    k = np.arange(n)
    mu = np.zeros(n)
    even = k % 2 == 0
    mu[even] = 2.0 / (1.0 - k[even].astype(float) ** 2)
    weights = mu @ Cmat
    D = np.empty((n, n))
    S = np.empty((n, n))
    for j in range(n):
        cj = Cmat[:, j]
        D[:, j] = C.chebval(nodes, C.chebder(cj))
        anti = C.chebint(cj)
        S[:, j] = C.chebval(nodes, anti) - C.chebval(-1.0, anti)
    for a in (nodes, weights, D, S):
        a.setflags(write=False)
    return nodes, weights, D, S


def fiber_geometry(X, p):
    """Host reference of the per-fiber geometry the device computes.

    Returns s, s_alpha, L, tangents for a (p+1,3) centerline (spectral.py:
    139-154, fiber.py:133-147).
    """
    nodes, w, D, S = grid(p)
    X = np.asarray(X, dtype=float)
    Xa = D @ X
    s_alpha = np.sqrt((Xa * Xa).sum(axis=1))
    if s_alpha.min() <= 1e-12:
        raise DegenerateFiberError("centerline parametrization is degenerate")
    anti = C.chebint(values_to_coeffs(s_alpha))
    s = C.chebval(nodes, anti) - C.chebval(-1.0, anti)
    return s, s_alpha, float(s[0]), Xa / s_alpha[:, None]


@functools.lru_cache(maxsize=None)
def coeff_matrix(p):
    """(n,n) map from nodal values to Chebyshev coefficients (DCT-I, as
    cheb_transform in spectral.py:37-50), column by column."""
    n = int(p) + 1
    eye = np.eye(n)
    Cm = np.stack([values_to_coeffs(eye[:, j]) for j in range(n)], axis=1)
    Cm.setflags(write=False)
    return Cm


# -- the reference's spectral API (spectral.py:37-154) on top of grid(p) ------

def cheb_transform(values):
    """Chebyshev coefficients of the interpolant through 1-d nodal values."""
    values = np.asarray(values, dtype=float)
    if values.ndim != 1 or values.size < 2:
        raise ValueError("expected a 1-d array of at least two nodal values")
    return values_to_coeffs(values)


def cheb_eval_nodes(coeffs, nodes):
    """Chebyshev series at the given points (Clenshaw)."""
    return C.chebval(nodes, coeffs)


def cheb_diff(values, grid_):
    """Nodal d/d(alpha) of the interpolant, via the coefficient recursion."""
    values = np.asarray(values, dtype=float)
    if values.size != grid_.p + 1:
        raise ValueError(f"expected {grid_.p + 1} nodal values, got {values.size}")
    return C.chebval(grid_.nodes, C.chebder(cheb_transform(values)))


def cheb_integrate(values, grid_):
    """Clenshaw-Curtis integral over [-1, 1]."""
    values = np.asarray(values, dtype=float)
    if values.size != grid_.p + 1:
        raise ValueError(f"expected {grid_.p + 1} nodal values, got {values.size}")
    return float(grid_.weights @ values)


def cheb_interp(values, alpha):
    """Barycentric evaluation of the interpolant at alpha in [-1, 1]."""
    values = np.asarray(values, dtype=float)
    if abs(alpha) > 1.0 + 1e-12:
        raise ValueError(f"interpolation point {alpha} outside [-1, 1]")
    alpha = min(1.0, max(-1.0, float(alpha)))
    p = values.size - 1
    d = alpha - cheb_nodes(p)
    hit = np.nonzero(np.abs(d) < 1e-15)[0]
    if hit.size:
        return float(values[hit[0]])
    w = np.where(np.arange(p + 1) % 2 == 0, 1.0, -1.0)
    w[0] *= 0.5
    w[-1] *= 0.5
    t = w / d
    return float((t @ values) / t.sum())


class ChebyshevGrid:
    """Order-p grid: nodes, Clenshaw-Curtis weights, dense D_alpha (spectral.py:114-136)."""

    def __init__(self, p):
        nodes, weights, D, _ = grid(p)
        self.p = int(p)
        self.nodes, self.weights, self.D = nodes, weights, D

    def __repr__(self):
        return f"ChebyshevGrid(p={self.p})"


def arclength_map(X, grid_):
    """(s, s_alpha, L) of a nodal centerline (spectral.py:139-154)."""
    X = np.asarray(X, dtype=float)
    if X.shape != (grid_.p + 1, 3):
        raise ValueError(f"expected centerline of shape ({grid_.p + 1}, 3)")
    s, s_alpha, L, _ = fiber_geometry(X, grid_.p)
    return s, s_alpha, L
