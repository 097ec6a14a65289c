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


def cheb_nodes(p):
    """Extremal points, symmetrised to be exactly antisymmetric (spectral.py:24-34)."""
    p = int(p)
    if p < 1:
        raise ValueError(f"order must be an integer >= 1, got {p}")
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
    p = int(p)
    if p < 4:
        raise ValueError(f"grid order must be an integer >= 4, got {p}")
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
        raise ValueError("centerline parametrization is degenerate")
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
