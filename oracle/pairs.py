"""ORACLE (test infrastructure only): ctypes binding of oracle_pairs.c.

Mirrors the reference's numba kernels one to one
(/root/reference/pkg/src/slenderflow/kernels.py), same names and return
values, computed on the CPU with OpenMP over targets.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle_pairs.so")

_lib = None
_D, _I64, _P = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        for name in ("or_stokeslet_sum", "or_doublet_sum"):
            getattr(L, name).argtypes = [_P, _P, _I64, _P, _P, _I64, _P, _D, _P]
            getattr(L, name).restype = _I64
        L.or_stresslet_sum.argtypes = [_P, _P, _I64, _P, _P, _I64, _P, _P, _D, _P]
        L.or_stresslet_sum.restype = _I64
        L.or_stresslet_sum_subtracted.argtypes = [_P, _P, _P, _P, _I64, _D, _P]
        L.or_stresslet_sum_subtracted.restype = None
        L.or_stresslet_rowsum.argtypes = [_P, _P, _P, _I64, _D, _P]
        L.or_stresslet_rowsum.restype = None
        L.or_kdelta_matrix.argtypes = [_P, _P, _P, _P, _P, _I64, _D, _D, _P]
        L.or_kdelta_matrix.restype = None
        L.or_kdelta_matrix_batched.argtypes = [_P, _P, _P, _P, _P, _I64, _I64, _P, _D, _P]
        L.or_kdelta_matrix_batched.restype = None
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def num_threads():
    return lib().or_num_threads()


def set_num_threads(n):
    lib().or_set_num_threads(int(n))


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    return a.ctypes.data if a.size else None


def stokeslet_sum(trg, tgrp, src, sgrp, f, pref):
    trg, src, f = _c(trg).reshape(-1, 3), _c(src).reshape(-1, 3), _c(f).reshape(-1, 3)
    tgrp, sgrp = _c(tgrp, np.int64), _c(sgrp, np.int64)
    out = np.zeros((trg.shape[0], 3))
    bad = lib().or_stokeslet_sum(_p(trg), _p(tgrp), trg.shape[0], _p(src), _p(sgrp),
                                 src.shape[0], _p(f), float(pref), _p(out))
    return out, int(bad)


def doublet_sum(trg, tgrp, src, sgrp, f, pref):
    trg, src, f = _c(trg).reshape(-1, 3), _c(src).reshape(-1, 3), _c(f).reshape(-1, 3)
    tgrp, sgrp = _c(tgrp, np.int64), _c(sgrp, np.int64)
    out = np.zeros((trg.shape[0], 3))
    bad = lib().or_doublet_sum(_p(trg), _p(tgrp), trg.shape[0], _p(src), _p(sgrp),
                               src.shape[0], _p(f), float(pref), _p(out))
    return out, int(bad)


def stresslet_sum(trg, tgrp, src, sgrp, nrm, qw, pref):
    trg, src = _c(trg).reshape(-1, 3), _c(src).reshape(-1, 3)
    nrm, qw = _c(nrm).reshape(-1, 3), _c(qw).reshape(-1, 3)
    tgrp, sgrp = _c(tgrp, np.int64), _c(sgrp, np.int64)
    out = np.zeros((trg.shape[0], 3))
    bad = lib().or_stresslet_sum(_p(trg), _p(tgrp), trg.shape[0], _p(src), _p(sgrp),
                                 src.shape[0], _p(nrm), _p(qw), float(pref), _p(out))
    return out, int(bad)


def stresslet_sum_subtracted(nodes, nrm, w, q, pref):
    nodes, nrm, q = _c(nodes).reshape(-1, 3), _c(nrm).reshape(-1, 3), _c(q).reshape(-1, 3)
    w = _c(w)
    out = np.zeros((nodes.shape[0], 3))
    lib().or_stresslet_sum_subtracted(_p(nodes), _p(nrm), _p(w), _p(q), nodes.shape[0],
                                      float(pref), _p(out))
    return out


def stresslet_rowsum(nodes, nrm, w, pref):
    nodes, nrm, w = _c(nodes).reshape(-1, 3), _c(nrm).reshape(-1, 3), _c(w)
    out = np.zeros((nodes.shape[0], 3, 3))
    lib().or_stresslet_rowsum(_p(nodes), _p(nrm), _p(w), nodes.shape[0], float(pref), _p(out))
    return out


def kdelta_matrix(X, s, s_alpha, tang, w, delta, pref):
    X, tang = _c(X).reshape(-1, 3), _c(tang).reshape(-1, 3)
    s, s_alpha, w = _c(s), _c(s_alpha), _c(w)
    n = X.shape[0]
    K = np.zeros((3 * n, 3 * n))
    lib().or_kdelta_matrix(_p(X), _p(s), _p(s_alpha), _p(tang), _p(w), n, float(delta),
                           float(pref), _p(K))
    return K


def kdelta_matrix_batched(X, s, s_alpha, tang, w, delta, pref):
    """(nf,n,3) fibers -> (nf,3n,3n); one reference call per fiber."""
    X, tang = _c(X), _c(tang)
    s, s_alpha, w, delta = _c(s), _c(s_alpha), _c(w), _c(delta)
    nf, n = X.shape[0], X.shape[1]
    K = np.zeros((nf, 3 * n, 3 * n))
    lib().or_kdelta_matrix_batched(_p(X), _p(s), _p(s_alpha), _p(tang), _p(w), nf, n, _p(delta),
                                   float(pref), _p(K))
    return K
