"""Device-resident fiber HI operator (the hot path of every GMRES matvec).

FiberHIOperator freezes one geometry on the B200 -- the layout the
reference's InteractionCache builds on the host every step
(system.py:492-562): fiber nodes as both targets and sources, fiber-id
groups, quadrature weights w s_alpha, doublet coefficients (eps L)^2/2,
the K_delta matrices and the near-field correction maps -- and applies

    u_nl   = complementary_velocities(...).fibers     system.py:623-709 (fiber part)
    u_self = local_mobility_apply + nonlocal_Kdelta_apply   fiber.py:244-258

to force densities that live on the device.  All arithmetic is in
libsf_b200.so; torch only carries the buffers and the stream.
"""

import ctypes
import math

import numpy as np

from . import _native, spectral
from ._native import SF_MODE_FP32C, SF_MODE_FP64


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class NearMap:
    """CSR (by target) of near-field correction maps W (3 x 3n) on the device.

    entries: iterable of (t, l, W) in the reference's list order
    (system.py:559-586); within a target the list order is preserved.
    """

    def __init__(self, entries, n_nodes, device):
        import torch
        entries = list(entries)
        self.count = len(entries)
        if not entries:
            self.nrows = 0
            self.row_ptr = self.rows = self.w_off = self.x_off = self.x_len = self.W = None
            return
        t = np.array([e[0] for e in entries], dtype=np.int64)
        l = np.array([e[1] for e in entries], dtype=np.int64)
        W = np.stack([np.asarray(e[2].cpu() if torch.is_tensor(e[2]) else e[2],
                                 dtype=float).reshape(3, -1) for e in entries])
        order = np.argsort(t, kind="stable")
        t, l, W = t[order], l[order], W[order]
        rows, starts = np.unique(t, return_index=True)
        row_ptr = np.append(starts, t.size).astype(np.int64)
        L = 3 * n_nodes
        dev = dict(device=device)
        self.nrows = rows.size
        self.row_ptr = torch.as_tensor(row_ptr, **dev)
        self.rows = torch.as_tensor(rows, **dev)
        self.w_off = torch.as_tensor(np.arange(t.size, dtype=np.int64) * 3 * L, **dev)
        self.x_off = torch.as_tensor(l * L, **dev)
        self.x_len = torch.full((t.size,), L, dtype=torch.int64, device=device)
        self.W = torch.as_tensor(np.ascontiguousarray(W), dtype=torch.float64, device=device)


class FiberHIOperator:
    """Frozen-geometry fiber HI operator on one device.

    X: (nf, n, 3) centrelines (numpy or torch); eps: scalar or (nf,);
    delta: None for the reference default 0.01 L (fiber.py:127,144), else
    scalar or (nf,) explicit regularisation lengths.
    """

    def __init__(self, X, eps, mu=1.0, include_doublet=True, near=(), delta=None,
                 device="cuda", mode=SF_MODE_FP64, shard=(0, 1)):
        import torch
        if mu <= 0:
            raise ValueError("viscosity must be positive")
        self.device = torch.device(device)
        dev = dict(dtype=torch.float64, device=self.device)
        X = torch.as_tensor(X, **dev).contiguous()
        if X.ndim != 3 or X.shape[2] != 3:
            raise ValueError("centrelines must be (n_fibers, n_nodes, 3)")
        nf, n, _ = X.shape
        self.nf, self.n, self.p = nf, n, n - 1
        self.N = nf * n
        self.mu = float(mu)
        self.mode = int(mode)
        self.X = X
        _, wcc, D, S = spectral.grid(self.p)
        self.wcc = torch.tensor(wcc, **dev)
        self.D = torch.tensor(D, **dev)
        self.S = torch.tensor(S, **dev)
        self.s = torch.empty((nf, n), **dev)
        self.s_alpha = torch.empty((nf, n), **dev)
        self.tang = torch.empty((nf, n, 3), **dev)
        self.wnode = torch.empty((nf, n), **dev)
        self.L = torch.empty(nf, **dev)
        if delta is None:
            self.delta = torch.empty(nf, **dev)
            ratio = 0.01
        else:
            self.delta = torch.as_tensor(np.broadcast_to(np.asarray(delta, dtype=float), (nf,)).copy(),
                                         **dev)
            ratio = -1.0
        degenerate = torch.zeros(1, dtype=torch.int32, device=self.device)
        st = _stream()
        _native.call("sf_fiber_geometry_batched", _ptr(X), nf, n, _ptr(self.D), _ptr(self.S),
                     _ptr(self.wcc), ratio, _ptr(self.s), _ptr(self.s_alpha), _ptr(self.tang),
                     _ptr(self.wnode), _ptr(self.L), _ptr(self.delta), _ptr(degenerate), st)
        if int(degenerate.item()):
            raise ValueError("centerline parametrization is degenerate")
        self.pref = 1.0 / (8.0 * math.pi * self.mu)
        # target-block shard: this rank owns fibers [f0, f0 + nown) as targets
        rank, world = shard
        self.rank, self.world = int(rank), int(world)
        per = -(-nf // self.world)
        self.f0 = min(nf, self.rank * per)
        self.nown = min(nf, self.f0 + per) - self.f0
        self.Nown = self.nown * n
        o = self.f0
        self.K = torch.empty((self.nown, 3 * n, 3 * n), **dev)
        _native.call("sf_kdelta_build_batched", _ptr(X[o:]), _ptr(self.s[o:]),
                     _ptr(self.s_alpha[o:]), _ptr(self.tang[o:]), _ptr(self.wcc), self.nown, n,
                     _ptr(self.delta[o:]), self.pref, _ptr(self.K), st)
        eps_np = np.broadcast_to(np.asarray(eps, dtype=float), (nf,)).copy()
        self.eps = torch.as_tensor(eps_np, **dev)
        self.c_log = torch.as_tensor(-np.log(eps_np ** 2 * math.e) / (8.0 * math.pi * self.mu),
                                     **dev)
        self.c_two = 2.0 / (8.0 * math.pi * self.mu)
        self.groups = torch.arange(nf, dtype=torch.int64,
                                   device=self.device).repeat_interleave(n).contiguous()
        if include_doublet:
            c = (self.eps * self.L) ** 2 / 2.0          # system.py:542
            self.dcoef = c.repeat_interleave(n).contiguous()
        else:
            self.dcoef = None
        lo, hi = self.f0 * n, (self.f0 + self.nown) * n
        own = [(t - lo, l, W) for t, l, W in near if lo <= t < hi]
        self.near = NearMap(own, n, self.device)
        self.bad = torch.zeros(1, dtype=torch.int64, device=self.device)

    # pair interactions evaluated by one apply on this shard (non-excluded pairs)
    @property
    def pairs_per_apply(self):
        return self.Nown * self.N - self.nown * self.n * self.n

    @property
    def symmetric(self):
        """Whether the fiber pair sum runs the symmetric evaluation
        (SF_MODE_FP64, whole system on this rank, >= 8192 points)."""
        import os
        return (self.mode in (SF_MODE_FP64, SF_MODE_FP32C) and self.world == 1 and self.N >= 8192
                and os.environ.get("SF_SYMMETRIC", "1") != "0")

    @property
    def symmetric_shard(self):
        """Multi-GPU form of the symmetric evaluation: this rank computes its
        share of the unit-pair tasks for ALL points; the dist layer sums the
        ranks' partials with a reduce-scatter."""
        import os
        return (self.mode in (SF_MODE_FP64, SF_MODE_FP32C) and self.world > 1 and self.N >= 8192
                and os.environ.get("SF_SYMMETRIC", "1") != "0")

    def task_ranges(self, world=None):
        """[(t0, count)] per rank of the symmetric unit-pair tasks, balanced
        by modelled cost (dist.task_ranges; computed once per geometry and
        world size, identically on every rank)."""
        from .dist import task_ranges
        world = self.world if world is None else world
        cache = self.__dict__.setdefault("_ranges", {})
        if world not in cache:
            cache[world] = task_ranges(self.X.reshape(-1, 3), self.groups, self.N, self.n,
                                       self.mode, world)
        return cache[world]

    @property
    def shard_pairs(self):
        """Non-excluded ordered pair interactions of this rank's task share."""
        t0, cnt = self.task_ranges()[self.rank]
        return int(_native.load().sf_sym_range_pairs(self.N, self.n, self.mode, t0, cnt))

    def symmetric_partial(self, f, out=None, rank=None, world=None):
        """(N,3) contribution of this rank's unit-pair tasks to every point
        (sf_sbt_symmetric_tasks over the rank's cost-balanced task range)."""
        import torch
        f = torch.as_tensor(f, dtype=torch.float64, device=self.device).contiguous()
        if out is None:
            out = torch.empty((self.N, 3), dtype=torch.float64, device=self.device)
        rank = self.rank if rank is None else rank
        t0, cnt = self.task_ranges(world)[rank]
        _native.call("sf_sbt_symmetric_tasks", _ptr(self.X), _ptr(self.groups), self.N, self.n,
                     _ptr(f), _ptr(self.wnode), _ptr(self.dcoef), self.pref, self.mode, t0, cnt,
                     _ptr(out), _ptr(self.bad), _stream())
        return out

    def finish_own(self, u_own, f, out_self=None, self_terms=True):
        """Near corrections and self terms of this rank's targets, after the
        pair sums of every rank were summed into u_own (Nown,3)."""
        import torch
        f = torch.as_tensor(f, dtype=torch.float64, device=self.device).reshape(-1, 3).contiguous()
        nm = self.near
        st = _stream()
        if nm.nrows:
            _native.call("sf_near_apply", _ptr(nm.row_ptr), _ptr(nm.rows), nm.nrows, _ptr(nm.w_off),
                         _ptr(nm.x_off), _ptr(nm.x_len), _ptr(nm.W), _ptr(f), _ptr(u_own), st)
        if self_terms:
            if out_self is None:
                out_self = torch.empty((self.Nown, 3), dtype=torch.float64, device=self.device)
            o = self.f0
            _native.call("sf_self_apply_batched", _ptr(self.K), _ptr(self.tang[o:]),
                         _ptr(self.c_log[o:]), self.c_two, _ptr(f[o * self.n:]), self.nown, self.n,
                         0, _ptr(out_self), st)
        return u_own, (out_self if self_terms else None)

    @property
    def launches_per_apply(self):
        """Kernels one apply launches: symmetric path = pack, slab meta, a
        task kernel and an ordered reduce per wave, final scale
        (sf_sym_launch_count); direct path = pack, tile meta, pair kernel
        (+ ordered split reduce); then near (if any) and self terms."""
        if self.symmetric:
            pair = _native.load().sf_sym_launch_count(self.N, self.n, self.mode, 0, 1)
        elif self.symmetric_shard:
            t0, cnt = self.task_ranges()[self.rank]
            pair = _native.load().sf_sym_range_launch_count(self.N, self.n, self.mode, t0, cnt)
        else:
            split = _native.load().sf_pair_split(self.Nown, self.N)
            pair = 3 + (1 if split > 1 else 0)
        return pair + (1 if self.near.nrows else 0) + 1

    def apply(self, f, out_nl=None, out_self=None, self_terms=True):
        """u_nl and u_self (each (Nown,3); u_self None if self_terms=False)
        for the force densities f (nf,n,3) of ALL fibers."""
        import torch
        f = torch.as_tensor(f, dtype=torch.float64, device=self.device).contiguous()
        if f.numel() != 3 * self.N:
            raise ValueError(f"expected {self.N} force vectors")
        if out_nl is None:
            out_nl = torch.empty((self.Nown, 3), dtype=torch.float64, device=self.device)
        if self_terms and out_self is None:
            out_self = torch.empty((self.Nown, 3), dtype=torch.float64, device=self.device)
        nm = self.near
        _native.call("sf_fiber_hi_apply", _ptr(self.X), _ptr(self.groups), self.nf, self.n,
                     self.f0, self.nown,
                     _ptr(self.wnode), _ptr(self.dcoef), self.pref, self.mode, _ptr(self.K),
                     _ptr(self.tang), _ptr(self.c_log), self.c_two, _ptr(nm.row_ptr),
                     _ptr(nm.rows), nm.nrows, _ptr(nm.w_off), _ptr(nm.x_off), _ptr(nm.x_len),
                     _ptr(nm.W), _ptr(f), _ptr(out_nl), _ptr(out_self if self_terms else None),
                     _ptr(self.bad), _stream())
        return out_nl, (out_self if self_terms else None)

    def check_bad(self):
        """Raise like the reference when a cross-group coincidence was skipped."""
        from .kernels import SingularEvaluationError
        if int(self.bad.item()):
            raise SingularEvaluationError("a target coincides with another fiber's node")
