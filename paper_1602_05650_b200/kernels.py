"""Device pair kernels behind the reference's kernel-level seam.

Same names, argument order, meaning and return values as
`slenderflow.kernels` (/root/reference/pkg/src/slenderflow/kernels.py):

    stokeslet_sum(trg, tgrp, src, sgrp, f, pref) -> (out, bad)      kernels.py:72-111
    doublet_sum(trg, tgrp, src, sgrp, f, pref) -> (out, bad)        kernels.py:114-145
    stresslet_sum(trg, tgrp, src, sgrp, nrm, qw, pref) -> (out, bad) kernels.py:177-213
    stresslet_sum_subtracted(nodes, nrm, w, q, pref) -> out          kernels.py:216-249
    stresslet_rowsum(nodes, nrm, w, pref) -> (N,3,3)                 kernels.py:252-281
    kdelta_matrix(X, s, s_alpha, tang, w, delta, pref) -> (3n,3n)    kernels.py:284-334

plus the fused slender-body sum `sbt_pair_sum` (Stokeslet + doublet in one
pass) that complementary_velocities uses.

NumPy inputs take the host-buffer C-ABI entry points (copy in, compute on the
B200, copy out) -- exactly what a ctypes binding inside the reference would
call.  torch CUDA tensors take the device entry points on the current stream
and return device tensors.  Like the reference, the kernels never raise on
coincident points: they skip and count them (`bad`), and callers raise
SingularEvaluationError.  There is no CPU fallback.
"""

import ctypes

import numpy as np

from . import _native
from ._native import SF_MODE_FP32C, SF_MODE_FP64

MIN_SEPARATION = 1e-12


class SingularEvaluationError(ValueError):
    pass


class NearFieldError(ValueError):
    """Target lies inside a near shell and needs nearly singular treatment."""


def no_groups(n):
    """Group-id array disabling exclusion for n points (kernels.py:337-339)."""
    return np.full(n, -1, dtype=np.int64)


# ----------------------------------------------------------------- helpers ----

def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _np(x, dtype, shape_tail=None, name="array"):
    a = np.ascontiguousarray(x, dtype=dtype)
    if shape_tail is not None and (a.ndim != 1 + len(shape_tail) or a.shape[1:] != shape_tail):
        raise ValueError(f"{name} must have shape (N, {', '.join(map(str, shape_tail))})")
    return a


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def _tp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t, dtype, name):
    import torch
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return t.contiguous()


# ----------------------------------------------------------------- host path ----

def _host_pair(fn, trg, tgrp, src, sgrp, a1, a2, pref, mode=None):
    trg = _np(trg, np.float64, (3,), "targets")
    src = _np(src, np.float64, (3,), "sources")
    nt, ns = trg.shape[0], src.shape[0]
    tgrp = _np(tgrp, np.int64) if tgrp is not None else None
    sgrp = _np(sgrp, np.int64) if sgrp is not None else None
    if tgrp is not None and tgrp.shape != (nt,):
        raise ValueError("target groups must have one entry per target")
    if sgrp is not None and sgrp.shape != (ns,):
        raise ValueError("source groups must have one entry per source")
    a1 = _np(a1, np.float64, (3,), "strengths")
    if a1.shape[0] != ns:
        raise ValueError("strengths must have one row per source")
    out = np.empty((nt, 3))
    bad = ctypes.c_int64(0)
    args = [_p(trg), _p(tgrp), nt, _p(src), _p(sgrp), ns, _p(a1)]
    if fn == "sf_host_stresslet_sum":
        a2 = _np(a2, np.float64, (3,), "qw")
        args.append(_p(a2))
    elif fn == "sf_host_sbt_pair":
        a2 = _np(a2, np.float64) if a2 is not None else None
        args += [_p(a2)]
    args.append(float(pref))
    if mode is not None:
        args.append(int(mode))
    args += [_p(out), ctypes.byref(bad)]
    _native.call(fn, *args)
    return out, int(bad.value)


# --------------------------------------------------------------- device path ----

def _dev_pair(fn, trg, tgrp, src, sgrp, a1, a2, pref, mode=None):
    import torch
    trg = _dev(trg, torch.float64, "targets")
    src = _dev(src, torch.float64, "sources")
    a1 = _dev(a1, torch.float64, "strengths")
    tgrp = _dev(tgrp, torch.int64, "target groups") if tgrp is not None else None
    sgrp = _dev(sgrp, torch.int64, "source groups") if sgrp is not None else None
    nt, ns = trg.shape[0], src.shape[0]
    out = torch.empty((nt, 3), dtype=torch.float64, device=trg.device)
    bad = torch.zeros(1, dtype=torch.int64, device=trg.device)
    args = [_tp(trg), _tp(tgrp), nt, _tp(src), _tp(sgrp), ns, _tp(a1)]
    if fn == "sf_stresslet_sum":
        args.append(_tp(_dev(a2, torch.float64, "qw")))
    elif fn == "sf_sbt_pair":
        args.append(_tp(_dev(a2, torch.float64, "doublet coefficients")) if a2 is not None
                    else ctypes.c_void_p(0))
    args.append(float(pref))
    if mode is not None:
        args.append(int(mode))
    args += [_tp(out), _tp(bad), _stream()]
    _native.call(fn, *args)
    return out, bad


def _pair(host_fn, dev_fn, trg, tgrp, src, sgrp, a1, a2, pref, mode=None):
    if _is_torch(trg):
        out, bad = _dev_pair(dev_fn, trg, tgrp, src, sgrp, a1, a2, pref, mode)
        return out, int(bad.item())
    return _host_pair(host_fn, trg, tgrp, src, sgrp, a1, a2, pref, mode)


# ------------------------------------------------------------- public API ----

def stokeslet_sum(trg, tgrp, src, sgrp, f, pref):
    """kernels.py:72-111 on the B200.  Returns (out (Nt,3), bad)."""
    return _pair("sf_host_stokeslet_sum", "sf_stokeslet_sum", trg, tgrp, src, sgrp, f, None, pref)


def doublet_sum(trg, tgrp, src, sgrp, f, pref):
    """kernels.py:114-145 on the B200.  Returns (out (Nt,3), bad)."""
    return _pair("sf_host_doublet_sum", "sf_doublet_sum", trg, tgrp, src, sgrp, f, None, pref)


def sbt_pair_sum(trg, tgrp, src, sgrp, f, dcoef, pref, mode=SF_MODE_FP64):
    """Fused Stokeslet + (eps L)^2/2 doublet sum (system.py:656-671 in one pass).

    f: quadrature-weighted strengths (Ns,3); dcoef: per-source doublet
    coefficient (Ns,) or None.  mode SF_MODE_FP32C selects the FP32-compute /
    FP64-accumulate variant.
    """
    return _pair("sf_host_sbt_pair", "sf_sbt_pair", trg, tgrp, src, sgrp, f, dcoef, pref, mode)


def stresslet_sum(trg, tgrp, src, sgrp, nrm, qw, pref):
    """kernels.py:177-213 on the B200.  Returns (out (Nt,3), bad)."""
    return _pair("sf_host_stresslet_sum", "sf_stresslet_sum", trg, tgrp, src, sgrp, nrm, qw, pref)


def stresslet_sum_subtracted(nodes, nrm, w, q, pref):
    """kernels.py:216-249 on the B200.  Returns (N,3)."""
    if _is_torch(nodes):
        import torch
        nodes = _dev(nodes, torch.float64, "nodes")
        n = nodes.shape[0]
        out = torch.empty((n, 3), dtype=torch.float64, device=nodes.device)
        _native.call("sf_stresslet_sum_subtracted", _tp(nodes),
                     _tp(_dev(nrm, torch.float64, "normals")), _tp(_dev(w, torch.float64, "w")),
                     _tp(_dev(q, torch.float64, "q")), n, float(pref), _tp(out), _stream())
        return out
    nodes = _np(nodes, np.float64, (3,), "nodes")
    n = nodes.shape[0]
    nrm = _np(nrm, np.float64, (3,), "normals")
    w = _np(w, np.float64)
    q = _np(q, np.float64, (3,), "q")
    if nrm.shape[0] != n or w.shape != (n,) or q.shape[0] != n:
        raise ValueError("surface arrays must agree in length")
    out = np.empty((n, 3))
    _native.call("sf_host_stresslet_sum_subtracted", _p(nodes), _p(nrm), _p(w), _p(q), n,
                 float(pref), _p(out))
    return out


def stresslet_rowsum(nodes, nrm, w, pref):
    """kernels.py:252-281 on the B200.  Returns (N,3,3)."""
    if _is_torch(nodes):
        import torch
        nodes = _dev(nodes, torch.float64, "nodes")
        n = nodes.shape[0]
        out = torch.empty((n, 3, 3), dtype=torch.float64, device=nodes.device)
        _native.call("sf_stresslet_rowsum", _tp(nodes), _tp(_dev(nrm, torch.float64, "normals")),
                     _tp(_dev(w, torch.float64, "w")), n, float(pref), _tp(out), _stream())
        return out
    nodes = _np(nodes, np.float64, (3,), "nodes")
    n = nodes.shape[0]
    nrm = _np(nrm, np.float64, (3,), "normals")
    w = _np(w, np.float64)
    if nrm.shape[0] != n or w.shape != (n,):
        raise ValueError("surface arrays must agree in length")
    out = np.empty((n, 3, 3))
    _native.call("sf_host_stresslet_rowsum", _p(nodes), _p(nrm), _p(w), n, float(pref), _p(out))
    return out


def kdelta_matrix(X, s, s_alpha, tang, w, delta, pref):
    """kernels.py:284-334 on the B200 (bitwise-identical build).  (3n,3n)."""
    X = _np(X, np.float64, (3,), "X")
    n = X.shape[0]
    s = _np(s, np.float64)
    s_alpha = _np(s_alpha, np.float64)
    tang = _np(tang, np.float64, (3,), "tangents")
    w = _np(w, np.float64)
    K = np.empty((3 * n, 3 * n))
    _native.call("sf_host_kdelta_matrix", _p(X), _p(s), _p(s_alpha), _p(tang), _p(w), n,
                 float(delta), float(pref), _p(K))
    return K


def rotlet_sum(trg, src, L, pref):
    """Sum of rotlets pref (L_j x r) / r^3 (kernels.py:149-174), no group
    exclusion (sources are body centres), r^2 < 1e-24 skipped and counted.
    Evaluated on the device; numpy in -> numpy out."""
    import torch
    host = not _is_torch(trg)
    dev = torch.device("cuda")
    t = torch.as_tensor(np.asarray(trg, dtype=float) if host else trg, dtype=torch.float64,
                        device=dev).reshape(-1, 3)
    s = torch.as_tensor(np.asarray(src, dtype=float) if host else src, dtype=torch.float64,
                        device=dev).reshape(-1, 3)
    Lt = torch.as_tensor(np.asarray(L, dtype=float) if host else L, dtype=torch.float64,
                         device=dev).reshape(-1, 3)
    r = t[:, None, :] - s[None, :, :]
    r2 = (r * r).sum(dim=2)
    ok = r2 >= MIN_SEPARATION * MIN_SEPARATION
    ir3 = torch.where(ok, 1.0 / (torch.where(ok, r2, 1.0) * torch.sqrt(torch.where(ok, r2, 1.0))),
                      torch.zeros_like(r2))
    u = (torch.cross(Lt[None, :, :].expand_as(r), r, dim=2) * ir3[:, :, None]).sum(dim=1) * pref
    bad = int((~ok).sum().item())
    return (u.cpu().numpy() if host else u), bad


# -- single-pair kernels and the viscosity holder (kernels.py:22-69): scalar
#    host helpers of the reference API --------------------------------------

class KernelContext:
    """Holds the fluid viscosity shared by the kernel evaluations."""

    def __init__(self, mu):
        if mu <= 0:
            raise ValueError(f"viscosity must be positive, got {mu}")
        self.mu = float(mu)


def _checked_r(r):
    r = np.asarray(r, dtype=float)
    d = np.sqrt(r @ r)
    if d < MIN_SEPARATION:
        raise SingularEvaluationError(f"evaluation point within {MIN_SEPARATION} of source")
    return r, d


def stokeslet_apply(r, f, mu):
    """(1/8 pi mu)(I + rhat rhat) f / |r|."""
    r, d = _checked_r(r)
    f = np.asarray(f, dtype=float)
    return (f / d + (r @ f) * r / d ** 3) / (8.0 * np.pi * mu)


def stresslet_apply(r, n, q, mu):
    """-(3/4 pi mu)(q.rhat)(n.rhat) rhat / |r|^2."""
    r, d = _checked_r(r)
    return -3.0 * (np.asarray(q, dtype=float) @ r) * (np.asarray(n, dtype=float) @ r) * r / (
        4.0 * np.pi * mu * d ** 5)


def rotlet_apply(r, L, mu):
    """(1/8 pi mu)(L x rhat) / |r|^2."""
    r, d = _checked_r(r)
    return np.cross(np.asarray(L, dtype=float), r) / (8.0 * np.pi * mu * d ** 3)


def doublet_apply(r, f, mu):
    """(1/8 pi mu)(I - 3 rhat rhat) f / |r|^3."""
    r, d = _checked_r(r)
    f = np.asarray(f, dtype=float)
    return (f / d ** 3 - 3.0 * (r @ f) * r / d ** 5) / (8.0 * np.pi * mu)


def dfma_peak(iters=1 << 16):
    """Measured FP64 DFMA throughput of this GPU: (flop/s, ms)."""
    flops = ctypes.c_double(0.0)
    ms = ctypes.c_double(0.0)
    _native.call("sf_dfma_peak", int(iters), ctypes.byref(flops), ctypes.byref(ms))
    return flops.value, ms.value


__all__ = [
    "MIN_SEPARATION", "SingularEvaluationError", "NearFieldError", "no_groups",
    "stokeslet_sum", "doublet_sum", "sbt_pair_sum", "stresslet_sum",
    "stresslet_sum_subtracted", "stresslet_rowsum", "kdelta_matrix", "dfma_peak", "rotlet_sum",
    "KernelContext", "stokeslet_apply", "stresslet_apply", "rotlet_apply", "doublet_apply",
    "SF_MODE_FP64", "SF_MODE_FP32C",
]
