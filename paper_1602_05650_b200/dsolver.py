"""Multi-GPU implicit step: sharded block rows, gathered GMRES.

One process per GPU.  Rank r owns a contiguous block of fibers (their X, T
unknowns and rows); rank 0 also owns the particle and periphery unknowns
(U, omega, q1, q0) and rows.

Per matvec:
  1. broadcast the surface/particle unknowns from rank 0;
  2. fiber force densities of the own fibers, all-gathered (NCCL) to all;
  3. particle wrenches: per-rank partial sums, all-reduced;
  4. fiber x fiber Stokeslet + doublet: the symmetric unit-pair tasks split
     over ranks + reduce-scatter (>= 8192 points), or own targets against
     all sources (direct);
  5. the other families (surface double layers, completion flow, near maps)
     for the rank's own targets; surface targets <- own fibers as per-rank
     partials, all-reduced; a large on-surface double layer split by its
     symmetric tasks and all-reduced;
  6. own fiber rows; surface rows on rank 0.
GMRES (default "gathered"): each iteration the ranks' rows of M A v are
all-gathered (one collective of the unknown-vector size) and every rank
runs the single-GPU GMRES on the full, identical vectors, so every rank
takes bitwise-identical Krylov decisions.  SF_DIST_GMRES=reduced instead
all-reduces every MGS inner product (one collective per inner product).
Errors that one rank detects (skipped pairs, singular fiber blocks) are
summed over the ranks first, so every rank raises together.

`Comm` hides the transport: TorchComm uses torch.distributed (NCCL on the
GPU box, gloo on the CPU), ThreadComm runs the ranks as threads on ONE GPU
(host-side barriers only; no kernel waits on another) for tests.
"""

import ctypes
import math
import os
import threading

import numpy as np

from . import _native, spectral
from .dist import shard_range
from .solver import (BC_CODES, LOG, FactorizationError, GmresParams, NonconvergenceError,
                     StepLayout, _kinetics_and_contacts, _precision_mode, _ptr,
                     _rotation_is_representable, _stream)
from .system import (ConfigurationError, SingularEvaluationError, FiberGeometry, InteractionCache, external_force_density,
                     stack_fibers)


# ------------------------------------------------------------------ comms ----
class TorchComm:
    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, group=self.group)
        return t

    def broadcast(self, t, src=0):
        self.dist.broadcast(t, src=src, group=self.group)
        return t

    def all_gather(self, out, inp):
        if self.nccl:
            self.dist.all_gather_into_tensor(out, inp, group=self.group)
        else:
            self.dist.all_gather(list(out.chunk(self.world)), inp, group=self.group)
        return out

    def reduce_scatter_sum(self, out, inp):
        if self.nccl:
            self.dist.reduce_scatter_tensor(out, inp, group=self.group)
        else:
            self.dist.all_reduce(inp, group=self.group)
            out.copy_(inp.chunk(self.world)[self.rank])
        return out


class ThreadHub:
    """Shared state of ThreadComm ranks (one process, one GPU)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm:
    """Collectives between threads of one process; sums in rank order."""

    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _exchange(self, t):
        import torch
        if t.is_cuda:
            torch.cuda.current_stream().synchronize()
        self.hub.slots[self.rank] = t
        self.hub.barrier.wait()
        return self.hub.slots

    def _done(self):
        import torch
        if self.hub.slots[self.rank].is_cuda:
            torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()

    def all_reduce_sum(self, t):
        slots = self._exchange(t.clone())
        acc = slots[0].clone()
        for k in range(1, self.world):
            acc += slots[k]
        self._done()
        t.copy_(acc)
        return t

    def broadcast(self, t, src=0):
        slots = self._exchange(t.clone())
        v = slots[src].clone()
        self._done()
        t.copy_(v)
        return t

    def all_gather(self, out, inp):
        slots = self._exchange(inp.clone())
        parts = [s.clone() for s in slots]
        self._done()
        for k, p in enumerate(parts):
            out.chunk(self.world)[k].copy_(p)
        return out

    def reduce_scatter_sum(self, out, inp):
        slots = self._exchange(inp.clone())
        acc = slots[0].chunk(self.world)[self.rank].clone()
        for k in range(1, self.world):
            acc += slots[k].chunk(self.world)[self.rank]
        self._done()
        out.copy_(acc)
        return out


# --------------------------------------------------------------- operator ----
class DistBlockOperator:
    """This rank's rows of the implicit step system (solver.py:187-364)."""

    def __init__(self, state, dt, comm, mu=None, symmetric=None, precision="fp64"):
        import torch
        if dt <= 0:
            raise ConfigurationError("time step must be positive")
        self.state, self.comm = state, comm
        self.dt = float(dt)
        self.mu = state.mu if mu is None else float(mu)
        self.layout = lay = StepLayout(state)
        self.device = dev = torch.device("cuda")
        f64 = dict(dtype=torch.float64, device=dev)
        nf = len(state.fibers)
        n = state.fibers[0].n_nodes if nf else 5
        if any(f.n_nodes != n for f in state.fibers):
            raise ConfigurationError("the distributed step needs one Chebyshev order for all "
                                     "fibers; mixed orders run on one GPU (solver.py)")
        self.nf, self.n = nf, n
        rank, world = comm.rank, comm.world
        self.f0, self.nown = shard_range(nf, rank, world)
        self.per = -(-nf // world) if nf else 0
        fo = lay.fib_off
        # target share: rank 0 [surfaces | own fibers], others own fibers
        n_surf_t = sum(p.mesh.n_nodes for p in state.particles) + \
            (state.periphery.mesh.n_nodes if state.periphery is not None else 0)
        self.n_surf_t = n_surf_t
        N = nf * n
        if symmetric is None:
            symmetric = N >= 8192 and os.environ.get("SF_SYMMETRIC", "1") != "0"
        self.symmetric = bool(symmetric) and nf > 0
        lo_f = n_surf_t + self.f0 * n
        hi_f = lo_f + self.nown * n
        ratios = [f.delta_ratio if f.delta_ratio is not None else -1.0 for f in state.fibers]
        deltas = [0.0 if f.delta_ratio is not None else f.delta for f in state.fibers]
        geo = FiberGeometry(stack_fibers(state.fibers), ratios, deltas, dev)
        self.geo = geo
        eps_all = torch.as_tensor([f.eps for f in state.fibers], **f64)
        self.fdcoef = ((eps_all * geo.L) ** 2 / 2.0).repeat_interleave(n).contiguous() \
            if nf else None
        self.fgrp = torch.as_tensor(np.repeat(np.arange(nf, dtype=np.int64), n), device=dev)
        # fiber targets: symmetric -> fiber pair sums come from the task split
        self.mode = _precision_mode(precision)
        self.cache_fib = (InteractionCache(state, target_range=(lo_f, hi_f), fiber_geometry=geo,
                                           fiber_pairs=not self.symmetric, mode=self.mode)
                          if self.nown else None)
        # surface targets: the fiber-source sums are split by fiber over the
        # ranks (each rank: surface targets <- its own fibers); the surface-
        # source sums, completion flows and near maps are split by target
        # (each rank: its slice of the surface targets); both land in one
        # (n_surf_t, 3) buffer and ONE all-reduce sums them for rank 0's rows.
        # Without fibers rank 0 evaluates every surface target itself.
        if n_surf_t and nf:
            per_t = -(-n_surf_t // world)
            a_t = min(n_surf_t, rank * per_t)
            self._surf_t_slice = (a_t, min(n_surf_t, a_t + per_t))
        else:
            self._surf_t_slice = (0, n_surf_t) if rank == 0 else (0, 0)
        a_t, b_t = self._surf_t_slice
        self.cache_surf = (InteractionCache(state, target_range=(a_t, b_t), fiber_geometry=geo,
                                            mode=self.mode, fiber_pairs=False)
                           if b_t > a_t else None)
        self._surf_part = None
        if n_surf_t and nf:
            tgt = np.vstack([p.mesh.nodes for p in state.particles]
                            + ([state.periphery.mesh.nodes] if state.periphery is not None else []))
            tgr = np.concatenate([np.full(p.mesh.n_nodes, nf + i, dtype=np.int64)
                                  for i, p in enumerate(state.particles)]
                                 + ([np.full(state.periphery.mesh.n_nodes, nf + len(state.particles),
                                             dtype=np.int64)] if state.periphery is not None else []))
            self._surf_trg = torch.as_tensor(tgt, **f64).contiguous()
            self._surf_tgrp = torch.as_tensor(tgr, device=dev)
            self._surf_part = torch.zeros((n_surf_t, 3), **f64)
            self._surf_bad = torch.zeros(1, dtype=torch.int64, device=dev)
        # frozen fiber operators of the OWN fibers
        o, no = self.f0, self.nown
        self.Dpow = torch.empty((no, 4, n, n), **f64)
        if no:
            _native.call("sf_fiber_dpow", _ptr(geo.D), _ptr(geo.s_alpha[o:]), no, n,
                         _ptr(self.Dpow), _stream())
        self.K = torch.empty((no, 3 * n, 3 * n), **f64)
        if no:
            _native.call("sf_kdelta_build_batched", _ptr(geo.X[o:]), _ptr(geo.s[o:]),
                         _ptr(geo.s_alpha[o:]), _ptr(geo.tang[o:]), _ptr(geo.wcc), no, n,
                         _ptr(geo.delta[o:]), 1.0 / (8.0 * math.pi * self.mu), _ptr(self.K),
                         _stream())
        own = state.fibers[o:o + no]
        eps = np.array([f.eps for f in own])
        self.E = torch.as_tensor(np.array([f.E for f in own], dtype=float), **f64)
        self.c_log = torch.as_tensor(-np.log(eps ** 2 * math.e) / (8.0 * math.pi * self.mu), **f64)
        self.c_two = 2.0 / (8.0 * math.pi * self.mu)
        self.Ldot = torch.as_tensor(np.array([f.Ldot for f in own], dtype=float), **f64)
        self.f_ext = (torch.as_tensor(np.ascontiguousarray(np.stack(
            [external_force_density(state, f) for f in own])), **f64)
            if (state.force_models and no) else None)
        kinds = np.zeros((no, 2), dtype=np.int32)
        par = np.zeros((no, 2, 12))
        body = np.full(no, -1, dtype=np.int32)
        for m, fib in enumerate(own):
            for e, bc in enumerate((fib.bc_plus, fib.bc_minus)):
                kinds[m, e] = BC_CODES[bc.kind]
                if bc.kind == "prescribedForceTorque":
                    par[m, e, 0:3], par[m, e, 3:6] = bc.force, bc.torque
                elif bc.kind == "hingedToSurface":
                    par[m, e, 6:9], par[m, e, 9] = bc.attachment, bc.stiffness
                elif bc.kind == "clampedToBody":
                    par[m, e, 10] = 0.0 if bc.tangent is None else 1.0
                    if e == 1:
                        body[m] = bc.body
        self.bc_kind = torch.as_tensor(kinds, device=dev)
        self.bc_par = torch.as_tensor(par, **f64)
        self.bc_body = torch.as_tensor(body, device=dev)
        np_ = len(state.particles)
        self.np = np_
        self.pcenter = (torch.as_tensor(np.stack([p.center for p in state.particles]), **f64)
                        if np_ else None)
        self.p_uoff = (torch.as_tensor(np.array([s.start for s in lay.U], dtype=np.int64), device=dev)
                       if np_ else None)
        self.ext = (torch.as_tensor(np.stack([np.concatenate([p.F_ext, p.L_ext])
                                              for p in state.particles]), **f64)
                    if (np_ and rank == 0) else None)
        self.nodes = torch.tensor(spectral.grid(n - 1)[0], **f64)
        self.sys = _native.FiberSys(
            nf=no, n=n, D=_ptr(geo.D), nodes=_ptr(self.nodes), Dpow=_ptr(self.Dpow),
            X=_ptr(geo.X[o:]), tang=_ptr(geo.tang[o:]), s_alpha=_ptr(geo.s_alpha[o:]),
            L=_ptr(geo.L[o:]), Ldot=_ptr(self.Ldot), E=_ptr(self.E), c_log=_ptr(self.c_log),
            c_two=self.c_two, K=_ptr(self.K), f_ext=_ptr(self.f_ext), bc_kind=_ptr(self.bc_kind),
            bc_par=_ptr(self.bc_par), bc_body=_ptr(self.bc_body), np=np_, pcenter=_ptr(self.pcenter),
            p_uoff=_ptr(self.p_uoff), fib_off=fo + 4 * n * o, dt=self.dt, mu=self.mu)
        # surfaces (rank 0 rows)
        # large meshes: the on-surface double layer is split over the ranks
        # (symmetric unit-pair tasks, sf_stresslet_sum_subtracted_partial)
        # and all-reduced; rank 0 consumes the sum in its surface rows
        self.dl_split = {}
        meshes = [(lay.q1[i], p.mesh) for i, p in enumerate(state.particles)]
        if state.periphery is not None:
            meshes.append((lay.q0, state.periphery.mesh))
        if os.environ.get("SF_SYMMETRIC", "1") != "0":
            for sl, m in meshes:
                if m.n_nodes >= 8192:
                    self.dl_split[sl.start] = dict(
                        sl=sl, n=m.n_nodes, nodes=torch.as_tensor(m.nodes, **f64),
                        nrm=torch.as_tensor(m.normals, **f64), w=torch.as_tensor(m.weights, **f64),
                        out=torch.empty((m.n_nodes, 3), **f64))
        self.surf = []
        # each surface's range in the surface-target list [particles | periphery]
        counts = [p.mesh.n_nodes for p in state.particles] + (
            [state.periphery.mesh.n_nodes] if state.periphery is not None else [])
        edges = np.concatenate([[0], np.cumsum(counts)]).astype(int)
        surf_slices = [slice(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
        if rank == 0:
            for i, part in enumerate(state.particles):
                m = part.mesh
                self.surf.append(dict(kind=0, pi=i, nodes=torch.as_tensor(m.nodes, **f64),
                                      nrm=torch.as_tensor(m.normals, **f64),
                                      w=torch.as_tensor(m.weights, **f64), n=m.n_nodes,
                                      area=m.area, center=self.pcenter[i], sl=lay.q1[i],
                                      uom=lay.U[i].start,
                                      tsl=surf_slices[i]))
            if state.periphery is not None:
                m = state.periphery.mesh
                self.surf.append(dict(kind=1, nodes=torch.as_tensor(m.nodes, **f64),
                                      nrm=torch.as_tensor(m.normals, **f64),
                                      w=torch.as_tensor(m.weights, **f64), n=m.n_nodes,
                                      area=m.area, center=None, sl=lay.q0, uom=None,
                                      tsl=surf_slices[-1]))
        # surface densities in cache order: (slice in u) for every surface, every rank
        self.dens_sl = list(lay.q1) + ([lay.q0] if lay.q0 is not None else [])
        # owned entries of the unknown vector: one contiguous range per rank
        # (rank 0's surface/particle block sits right before its fibers)
        lo = 0 if rank == 0 else fo + 4 * n * o
        self.own_lo, self.own_hi = lo, fo + 4 * n * (o + no)
        self.owned = [(self.own_lo, self.own_hi)] if self.own_hi > self.own_lo else []
        # scratch
        self._f_pad = torch.zeros((max(self.per, 1) * n, 3), **f64)
        self._f_full = torch.zeros((world * max(self.per, 1) * n, 3), **f64)
        self._wf = torch.empty((max(no, 1), 6), **f64)
        self._wr = torch.empty((max(np_, 1), 6), **f64)
        self._work = torch.empty(16, **f64)
        self._part = torch.empty((N, 3), **f64) if self.symmetric else None
        self._rs_in = torch.zeros((world * max(self.per, 1) * n, 3), **f64)
        self._rs_out = torch.zeros((max(self.per, 1) * n, 3), **f64)
        self._bad = torch.zeros(1, dtype=torch.int64, device=dev)
        self._checked = False
        self._task_range = None
        self.fiber_blocks = torch.empty((no, 4 * n, 4 * n), **f64)
        if no:
            _native.call("sf_fiber_self_blocks", ctypes.byref(self.sys), _ptr(self.fiber_blocks),
                         _stream())
        self.matvecs = 0

    @property
    def shape(self):
        return (self.layout.size, self.layout.size)

    def rows_device(self, u, constants, out=None):
        import torch
        c = self.comm
        st = _stream()
        n, fo, no = self.n, self.layout.fib_off, self.nown
        if out is None:
            out = torch.zeros_like(u)
        if fo:
            c.broadcast(u[:fo], src=0)               # U, omega, q1, q0 from rank 0
        sysp = ctypes.byref(self.sys)
        # own fiber forces -> all fibers
        self._f_pad.zero_()
        if no:
            _native.call("sf_fiber_forces", sysp, _ptr(u), int(constants), _ptr(self._f_pad), st)
        c.all_gather(self._f_full, self._f_pad)
        N = self.nf * n
        f_full = self._f_full[:N].contiguous()
        # particle wrenches: partial sums over own fibers, all-reduced
        if self.np:
            if no:
                _native.call("sf_particle_wrenches", sysp, _ptr(u), _ptr(self.ext), int(constants),
                             _ptr(self._wf), _ptr(self._wr), st)
            else:
                self._wr.zero_()
                if self.ext is not None and constants:
                    self._wr[:self.np].copy_(self.ext)
            c.all_reduce_sum(self._wr)
        q = (torch.cat([u[sl] for sl in self.dens_sl]).reshape(-1, 3) if self.dens_sl else None)
        wr = self._wr[:self.np] if self.np else None
        # fiber targets: the other families (and the fiber pairs when direct)
        # skipped-pair counts are geometric: checked on the first application only
        # skipped-pair counts depend only on the frozen geometry: they are
        # checked once, on the first application, collectively (_check_once)
        first = not self._checked
        ub_f = self.cache_fib.apply(f_full, q, wr, check=False) if no else None
        if self.symmetric:
            g = self.geo
            if self._task_range is None:      # cost-balanced split, once per geometry
                from .dist import task_ranges
                self._task_range = task_ranges(g.X.reshape(-1, 3), self.fgrp, N, n, self.mode,
                                               c.world)[c.rank]
            t0, cnt = self._task_range
            _native.call("sf_sbt_symmetric_tasks", _ptr(g.X), _ptr(self.fgrp), N, n,
                         _ptr(f_full), _ptr(g.wnode), _ptr(self.fdcoef),
                         1.0 / (8.0 * math.pi * self.mu), self.mode, t0, cnt,
                         _ptr(self._part), _ptr(self._bad), st)
            self._rs_in[:N].copy_(self._part)
            c.reduce_scatter_sum(self._rs_out, self._rs_in)
            if no:
                ub_f = ub_f + self._rs_out[:no * n]
        if no:
            _native.call("sf_fiber_rows", sysp, _ptr(u), _ptr(self._f_pad), _ptr(ub_f),
                         int(constants), _ptr(out), st)
        # surface targets <- own fibers, summed over ranks
        if self._surf_part is not None:
            if no:
                lo, hi = self.f0 * n, (self.f0 + no) * n
                sw = (self.geo.wnode.reshape(-1)[lo:hi, None] * f_full[lo:hi]).contiguous()
                _native.call("sf_sbt_pair", _ptr(self._surf_trg), _ptr(self._surf_tgrp),
                             self.n_surf_t, _ptr(self.geo.X.reshape(-1, 3)[lo:hi]),
                             _ptr(self.fgrp[lo:hi]), hi - lo, _ptr(sw), _ptr(self.fdcoef[lo:hi]),
                             1.0 / (8.0 * math.pi * self.mu), self.mode, _ptr(self._surf_part),
                             _ptr(self._surf_bad), st)
            else:
                self._surf_part.zero_()
            if self.cache_surf is not None:       # this rank's slice of the surface targets
                a_t, b_t = self._surf_t_slice
                self._surf_part[a_t:b_t] += self.cache_surf.apply(f_full, q, wr, check=False)
            c.all_reduce_sum(self._surf_part)
        pref_dl = -3.0 / (4.0 * math.pi * self.mu)
        for d in self.dl_split.values():
            _native.call("sf_stresslet_sum_subtracted_partial", _ptr(d["nodes"]), _ptr(d["nrm"]),
                         _ptr(d["w"]), _ptr(u[d["sl"]]), d["n"], pref_dl, c.rank, c.world,
                         _ptr(d["out"]), st)
            c.all_reduce_sum(d["out"])
        # surfaces (rank 0)
        if self.surf:
            ub_s = (self._surf_part if self._surf_part is not None
                    else self.cache_surf.apply(f_full, q, wr, check=False))
            for s in self.surf:
                qs = u[s["sl"]]
                rows = out[s["sl"]]
                if s["sl"].start in self.dl_split:
                    rows.copy_(self.dl_split[s["sl"].start]["out"].reshape(-1))
                else:
                    _native.call("sf_stresslet_sum_subtracted", _ptr(s["nodes"]), _ptr(s["nrm"]),
                                 _ptr(s["w"]), _ptr(qs), s["n"], pref_dl, _ptr(rows), st)
                ub = ub_s[s["tsl"]]
                if s["kind"] == 0:
                    _native.call("sf_wrench_flow", _ptr(s["nodes"]), s["n"], _ptr(s["center"]),
                                 _ptr(self._wr[s["pi"]]), self.mu, _ptr(rows), st)
                    uom = u[s["uom"]:s["uom"] + 6]
                    _native.call("sf_surface_rows", 0, _ptr(s["nodes"]), _ptr(s["nrm"]),
                                 _ptr(s["w"]), s["n"], _ptr(s["center"]), s["area"], _ptr(qs),
                                 _ptr(ub), _ptr(uom), self.mu, _ptr(self._work), _ptr(rows),
                                 _ptr(out[s["uom"]:s["uom"] + 6]), st)
                else:
                    _native.call("sf_surface_rows", 1, _ptr(s["nodes"]), _ptr(s["nrm"]),
                                 _ptr(s["w"]), s["n"], None, s["area"], _ptr(qs), _ptr(ub), None,
                                 self.mu, _ptr(self._work), _ptr(rows), None, st)
        if first:
            self._check_once()
        self.matvecs += 1
        return out

    def _check_once(self):
        """The skipped-pair counters of the first application (fiber targets,
        the symmetric task share, surface targets <- own fibers, surface
        targets), summed over the ranks in one collective, so that a
        coincidence on any rank raises SingularEvaluationError on every rank
        instead of leaving the others blocked in the next collective."""
        import torch
        flags = torch.zeros(6, dtype=torch.float64, device=self.device)
        if self.nown:
            flags[0:3] = self.cache_fib.bad.to(torch.float64)
        if self.symmetric:
            flags[3] = self._bad.to(torch.float64)[0]
        if self._surf_part is not None and self.nown:
            flags[4] = self._surf_bad.to(torch.float64)[0]
        if self.cache_surf is not None:
            flags[5] = self.cache_surf.bad.to(torch.float64).sum()
        self.comm.all_reduce_sum(flags)
        self._checked = True
        f = flags.cpu().numpy()
        if f[0] or f[3] or f[4]:
            raise SingularEvaluationError("a target coincides with another fiber's node")
        if f[1] or f[5]:
            raise SingularEvaluationError("a target coincides with another surface's node")
        if f[2]:
            raise SingularEvaluationError("target at a particle center")

    def rhs_device(self):
        import torch
        zero = torch.zeros(self.layout.size, dtype=torch.float64, device=self.device)
        return -self.rows_device(zero, True)


class DistPreconditioner:
    """Own fiber blocks (equilibrated LU) + surface diagonal on rank 0.

    body_coupling=True adds the body-coupled correction of
    solver.Preconditioner (not in the reference): the rigid particles'
    blocks inverted together with their coupling to the fibers, by the same
    Schur complement / Woodbury construction.  Distributed: W = D^-1
    A[f, U omega] for the OWN fibers only (fiber rows are fiber-local); the
    particle rows' dependence on the fiber unknowns, A[p, f] z, from the own
    fibers' force densities (all-gathered) and attachment wrenches
    (all-reduced), evaluated redundantly on every rank at the particle nodes
    (a target-ranged InteractionCache); S^-1 (pend x pend) redundant on every
    rank.  Per apply: one all-gather of fiber force densities, one
    all-reduce of the particle wrenches, one broadcast of the particle rows
    of v; the gathered GMRES variant only."""

    def __init__(self, op, body_coupling=False):
        import torch
        f64 = dict(dtype=torch.float64, device=op.device)
        self.op = op
        no, n = op.nown, op.n
        m = 4 * n
        self.m = m
        if m > 256:
            raise ConfigurationError("the distributed preconditioner factors blocks up to 4n = 256")
        self.off0 = op.layout.fib_off + 4 * n * op.f0
        st = _stream()
        self.LU = self.r = self.c = self.piv = None
        if no:
            A = op.fiber_blocks.clone()
            self.r = torch.empty((no, m), **f64)
            self.c = torch.empty((no, m), **f64)
            self.piv = torch.empty((no, m), dtype=torch.int32, device=op.device)
            info = torch.empty(no, dtype=torch.int32, device=op.device)
            _native.call("sf_block_lu", _ptr(A), no, m, _ptr(self.r), _ptr(self.c),
                         _ptr(self.piv), _ptr(info), st)
            self.LU = A
        # failed factorizations counted over every rank (one collective), so
        # all ranks raise together
        nbad = torch.zeros(1, **f64)
        if no:
            nbad[0] = (info > 0).sum().to(torch.float64)
        op.comm.all_reduce_sum(nbad)
        if float(nbad.item()) > 0:
            raise FactorizationError(f"{int(nbad.item())} fiber self-block(s) are not invertible")
        fo = op.layout.fib_off
        self.ndiag = fo if op.comm.rank == 0 else 0
        self.diag = torch.ones(max(self.ndiag, 1), **f64)
        pref = -3.0 / (4.0 * math.pi * op.mu)
        for s in op.surf:
            rs = torch.empty((s["n"], 3, 3), **f64)
            _native.call("sf_stresslet_rowsum", _ptr(s["nodes"]), _ptr(s["nrm"]), _ptr(s["w"]),
                         s["n"], pref, _ptr(rs), st)
            d = -torch.diagonal(rs, dim1=1, dim2=2)
            if s["kind"] == 1:
                d = d + 1.0 / op.mu + (s["nrm"] ** 2) * s["w"][:, None] / (op.mu * s["area"])
            self.diag[s["sl"]] = d.reshape(-1)
        self.coupled = None
        if body_coupling and op.np and op.nf:
            self._setup_body_coupling(op)

    # -- body coupling -----------------------------------------------------------
    def _setup_body_coupling(self, op):
        import torch

        from .solver import BlockOperator, _particle_block_inverse
        lay = op.layout
        c = op.comm
        f64 = dict(dtype=torch.float64, device=op.device)
        n, no, nsize = op.n, op.nown, lay.size
        pend = lay.q1[-1].stop
        npn = sum(p.mesh.n_nodes for p in op.state.particles)
        # particle-node targets against every fiber source (redundant per rank)
        pc = InteractionCache(op.state, target_range=(0, npn), fiber_geometry=op.geo, mode=op.mode)
        psurf = []
        for i, part in enumerate(op.state.particles):
            m = part.mesh
            psurf.append(dict(kind=0, pi=i, nodes=torch.as_tensor(m.nodes, **f64),
                              nrm=torch.as_tensor(m.normals, **f64),
                              w=torch.as_tensor(m.weights, **f64), n=m.n_nodes, area=m.area,
                              center=op.pcenter[i], sl=lay.q1[i], uom=lay.U[i].start,
                              tsl=pc.particle_slices[i]))
        self._pc, self._psurf, self._pend = pc, psurf, pend
        self._pq0 = torch.zeros((max(npn, 1), 3), **f64)
        self._pu0 = torch.zeros(6, **f64)
        self._pubar = torch.empty((max(npn, 1), 3), **f64)
        self._prow = torch.empty(pend, **f64)
        self._pwr = torch.empty((op.np, 6), **f64)
        self._pwork = torch.empty(16, **f64)
        lo = lay.fib_off + 4 * n * op.f0          # own fiber block range
        hi = lo + 4 * n * no
        self._own = (lo, hi)
        cols = [k for i in range(op.np) for k in range(lay.U[i].start, lay.U[i].start + 6)]
        # W = D^-1 A[f, U omega] on the own fibers: clamped ends see U, omega;
        # U, omega are no flow sources, so the fiber rows take ubar = 0
        zero_ubar = torch.zeros((max(no * n, 1), 3), **f64)
        W = torch.zeros((hi - lo, len(cols)), **f64)
        e = torch.zeros(nsize, **f64)
        rows = torch.zeros(nsize, **f64)
        z = torch.zeros(nsize, **f64)
        st = _stream()
        for k, j in enumerate(cols):
            if no:
                e[j] = 1.0
                _native.call("sf_fiber_rows", ctypes.byref(op.sys), _ptr(e), None, _ptr(zero_ubar),
                             0, _ptr(rows), st)
                e[j] = 0.0
                _native.call("sf_precond_apply", _ptr(self.LU), _ptr(self.r), _ptr(self.c),
                             _ptr(self.piv), no, self.m, self.off0, None, 0, _ptr(rows), _ptr(z), st)
                W[:, k] = z[lo:hi]
        # Z = A[p, f] W (collectives inside, every rank in the same order)
        Z = torch.empty((pend, len(cols)), **f64)
        t = torch.zeros(nsize, **f64)
        for k in range(len(cols)):
            t[lo:hi] = W[:, k]
            Z[:, k] = self._particle_rows(t)
        adapter = _ParticleBlocks(psurf, lay, op.device, op.mu, BlockOperator)
        Ainv = _particle_block_inverse(adapter)
        colt = torch.as_tensor(cols, device=op.device)
        AZ = Ainv @ Z
        C = torch.eye(len(cols), **f64) - AZ[colt]
        Cinv, info = torch.linalg.inv_ex(C)
        ok = torch.tensor([float(int(info.item()) == 0 and bool(torch.isfinite(Cinv).all()))],
                          **f64)
        c.all_reduce_sum(ok)                      # every rank raises together
        if float(ok.item()) < c.world:
            raise FactorizationError("particle Schur complement is singular")
        Sinv = torch.addmm(Ainv, AZ, Cinv @ Ainv[colt])
        self.coupled = dict(W=W, Sinv=Sinv, cols=colt)

    def _particle_rows(self, u):
        """A[particle rows, fiber columns] u from the fiber entries of u this
        rank owns (solver.BlockOperator.particle_rows_device, distributed)."""
        op, c = self.op, self.op.comm
        st = _stream()
        no = op.nown
        sysp = ctypes.byref(op.sys)
        op._f_pad.zero_()
        self._pwr.zero_()
        if no:
            _native.call("sf_fiber_forces", sysp, _ptr(u), 0, _ptr(op._f_pad), st)
            _native.call("sf_particle_wrenches", sysp, _ptr(u), None, 0, _ptr(op._wf),
                         _ptr(self._pwr), st)
        c.all_gather(op._f_full, op._f_pad)
        c.all_reduce_sum(self._pwr)
        f_full = op._f_full[:op.nf * op.n].contiguous()
        ubar = self._pc.apply(f_full, self._pq0, self._pwr, out=self._pubar, check=False)
        out = self._prow
        out.zero_()
        for s in self._psurf:
            rows = out[s["sl"]]
            _native.call("sf_wrench_flow", _ptr(s["nodes"]), s["n"], _ptr(s["center"]),
                         _ptr(self._pwr[s["pi"]]), op.mu, _ptr(rows), st)
            _native.call("sf_surface_rows", 0, _ptr(s["nodes"]), _ptr(s["nrm"]), _ptr(s["w"]),
                         s["n"], _ptr(s["center"]), s["area"], _ptr(self._pq0[:s["n"]]),
                         _ptr(ubar[s["tsl"]]), _ptr(self._pu0), op.mu, _ptr(self._pwork),
                         _ptr(rows), _ptr(out[s["uom"]:s["uom"] + 6]), st)
        return out

    def apply_device(self, v, out=None):
        import torch
        if out is None:
            out = torch.zeros_like(v)
        _native.call("sf_precond_apply", _ptr(self.LU), _ptr(self.r), _ptr(self.c), _ptr(self.piv),
                     self.op.nown, self.m, self.off0, _ptr(self.diag), self.ndiag, _ptr(v),
                     _ptr(out), _stream())
        cp = self.coupled
        if cp is not None:
            pend = self._pend
            vp = v[:pend].clone()
            self.op.comm.broadcast(vp, src=0)          # particle rows live on rank 0
            r = vp - self._particle_rows(out)
            zb = torch.mv(cp["Sinv"], r)
            out[:pend] = zb
            lo, hi = self._own
            if hi > lo:
                out[lo:hi].addmv_(cp["W"], zb[cp["cols"]], alpha=-1.0)
        return out


class _ParticleBlocks:
    """What solver._particle_block_inverse needs of an operator: the particle
    surface records, the layout, device and viscosity, and the dense own-
    particle block A[p, p] (BlockOperator.particle_block_matrix)."""

    def __init__(self, surf, layout, device, mu, block_operator_cls):
        self.surf, self.layout, self.device, self.mu = surf, layout, device, mu
        self._cls = block_operator_cls

    def particle_block_matrix(self):
        return self._cls.particle_block_matrix(self)


# ----------------------------------------------------------------- GMRES ----
class _GatheredOperator:
    """M A v with the ranks' owned rows all-gathered into the full vector, so
    every rank runs the single-GPU GMRES (fused MGS, deterministic dots) on
    identical full vectors: one collective per iteration instead of one per
    inner product, and bitwise-identical Krylov decisions on every rank."""

    def __init__(self, op, prec):
        import torch
        self.op, self.prec, self.comm = op, prec, op.comm
        self.device = op.device
        lay = op.layout
        self.n = lay.size
        spans = []
        for r in range(self.comm.world):
            f0, no = shard_range(op.nf, r, self.comm.world)
            lo = 0 if r == 0 else lay.fib_off + 4 * op.n * f0
            spans.append((lo, lay.fib_off + 4 * op.n * (f0 + no)))
        self.spans = spans
        self.width = max(max(b - a for a, b in spans), 1)
        f64 = dict(dtype=torch.float64, device=self.device)
        self._send = torch.zeros(self.width, **f64)
        self._recv = torch.zeros(self.comm.world * self.width, **f64)

    def gather(self, v_own):
        """Full vector from each rank's owned range of v_own."""
        import torch
        a, b = self.spans[self.comm.rank]
        self._send[:b - a].copy_(v_own[a:b])
        self.comm.all_gather(self._recv, self._send)
        full = torch.empty(self.n, dtype=torch.float64, device=self.device)
        for r, (lo, hi) in enumerate(self.spans):
            full[lo:hi].copy_(self._recv[r * self.width:r * self.width + hi - lo])
        return full

    def apply_device(self, v):
        return self.gather(self.prec.apply_device(self.op.rows_device(v, False)))


def dist_gmres_solve(op, prec, rhs, params=None, variant="gathered"):
    """Distributed GMRES (solver.py:444-516).

    "gathered" (default): the preconditioned matvec's owned rows are
    all-gathered and every rank runs solver.gmres_solve on the full vectors
    (one all-gather per iteration).  "reduced": every inner product is a
    local dot over the owned range plus an all-reduce of the scalar (k + 3
    collectives per iteration; kept for comparison)."""
    if variant == "gathered":
        from .solver import gmres_solve
        g = _GatheredOperator(op, prec)
        b = g.gather(prec.apply_device(rhs))
        return gmres_solve(g, None, b, params)
    return _dist_gmres_reduced(op, prec, rhs, params)


def _dist_gmres_reduced(op, prec, rhs, params=None):
    """solver.gmres_solve (solver.py:444-516) over the ranks' owned entries.
    Every inner product is a local deterministic dot over the rank's range
    plus an in-place all-reduce of the scalar, stream-ordered (NCCL), so the
    modified Gram-Schmidt loop needs no host sync; the Hessenberg column
    comes to the host once per iteration."""
    import torch
    if params is None:
        params = GmresParams()
    comm = op.comm
    dev = op.device
    n = rhs.numel()
    lo, hi = op.own_lo, op.own_hi
    work = torch.empty(296, dtype=torch.float64, device=dev)
    st = _stream()
    R = params.restart
    hcol = torch.zeros(R + 2, dtype=torch.float64, device=dev)
    scal = torch.zeros(1, dtype=torch.float64, device=dev)

    def dot_into(x, y, out, root=False):
        if hi > lo:
            _native.call("sf_dot", _ptr(x[lo:hi]), _ptr(y[lo:hi]), hi - lo, _ptr(work), _ptr(out),
                         0, st)
        else:
            out.zero_()
        comm.all_reduce_sum(out)
        if root:
            out.sqrt_()

    def M(v):
        return prec.apply_device(v)

    def A(v):
        return op.rows_device(v, False)

    b = M(rhs)
    dot_into(b, b, scal, root=True)
    beta0 = float(scal.item())
    if beta0 == 0.0:
        return torch.zeros(n, dtype=torch.float64, device=dev), 0, [0.0]
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    V = torch.zeros((R + 1, n), dtype=torch.float64, device=dev)
    history, iters = [], 0
    while True:
        r = b - M(A(x)) if iters else b
        dot_into(r, r, scal, root=True)
        beta = float(scal.item())
        if beta / beta0 <= params.tolerance:
            return x, iters, history or [beta / beta0]
        V[0].copy_(r / beta)
        H = np.zeros((R + 1, R))
        cs, sn, g = np.zeros(R), np.zeros(R), np.zeros(R + 1)
        g[0] = beta
        k = 0
        while k < R and iters < params.max_iterations:
            w = M(A(V[k])).contiguous()
            dot_into(w, w, hcol[R + 1:R + 2], root=True)               # wnorm
            for j in range(k + 1):                                       # modified Gram-Schmidt
                dot_into(V[j], w, hcol[j:j + 1])
                _native.call("sf_axpy_dev", _ptr(hcol[j:j + 1]), -1.0, 0, _ptr(V[j]), _ptr(w), n, st)
            dot_into(w, w, hcol[k + 1:k + 2], root=True)
            hh = hcol.cpu().numpy()
            wnorm = float(hh[R + 1])
            H[:k + 2, k] = hh[:k + 2]
            for j in range(k):
                tmp = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
                H[j, k] = tmp
            denom = math.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / denom if denom else 1.0
            sn[k] = H[k + 1, k] / denom if denom else 0.0
            H[k, k] = denom
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            iters += 1
            rel = abs(g[k + 1]) / beta0
            history.append(rel)
            breakdown = H[k + 1, k] <= 1e-12 * max(wnorm, 1e-300)
            if not breakdown:
                _native.call("sf_axpy_dev", _ptr(hcol[k + 1:k + 2]), 1.0, 2, _ptr(w), _ptr(V[k + 1]),
                             n, st)
            k += 1
            if rel <= params.tolerance or breakdown:
                break
        if k:
            y = np.linalg.solve(np.triu(H[:k, :k]), g[:k])
            coef = torch.as_tensor(y, dtype=torch.float64, device=dev)
            _native.call("sf_combine", _ptr(V), n, k, _ptr(coef), _ptr(x), n, st)
        rel = history[-1] if history else 0.0
        if rel <= params.tolerance:
            return x, iters, history
        if iters >= params.max_iterations:
            raise NonconvergenceError(
                f"GMRES did not reach {params.tolerance:g} within {params.max_iterations} "
                f"iterations (residual {rel:.3e})", best=x, iterations=iters, residuals=history)


def dist_backward_euler_step(state, dt, comm, params=None, return_info=False, symmetric=None,
                             precision="fp64", dt_min=None, body_coupling=False):
    """backward_euler_step (solver.py:528-592) over `comm`'s ranks: the same
    dt halving on NonconvergenceError down to dt_min (every rank takes the
    same GMRES decisions, so every rank retries together) and the same
    rotation check for non-spherical particles before any state changes.
    body_coupling=True selects the body-coupled preconditioner
    (DistPreconditioner; not in the reference).  The host state is
    replicated; every rank ends with the same state."""
    import torch
    if dt <= 0:
        raise ConfigurationError("time step must be positive")
    if dt_min is None:
        dt_min = dt / 64.0
    attempt = float(dt)
    variant = os.environ.get("SF_DIST_GMRES", "gathered")
    while True:
        op = DistBlockOperator(state, attempt, comm, symmetric=symmetric, precision=precision)
        rhs = op.rhs_device()
        if body_coupling and variant != "gathered":
            raise ConfigurationError("the body-coupled preconditioner needs SF_DIST_GMRES=gathered")
        prec = DistPreconditioner(op, body_coupling=body_coupling)
        try:
            x, iters, history = dist_gmres_solve(op, prec, rhs, params, variant=variant)
            break
        except NonconvergenceError as err:
            LOG.warning("step_rejected time=%.9g dt=%.3e residual=%.3e",
                        state.time, attempt, err.residuals[-1])
            if attempt / 2.0 < dt_min:
                raise
            attempt /= 2.0
    if variant != "gathered":
        # assemble the full solution on every rank: owned ranges summed (others 0)
        full = torch.zeros_like(x)
        for a, b in op.owned:
            full[a:b] = x[a:b]
        comm.all_reduce_sum(full)
        x = full
    sol = x.cpu().numpy()
    parts = op.layout.unpack(sol)
    for i, part in enumerate(state.particles):
        if not _rotation_is_representable(part, parts.omega[i], attempt):
            raise ConfigurationError("rotation of a non-spherical particle is not supported")
    for i, part in enumerate(state.particles):
        part.U = parts.U[i].copy()
        part.omega = parts.omega[i].copy()
        part.q = parts.q1[i].copy()
        part.translate(attempt * part.U)
    if state.periphery is not None:
        state.periphery.q = parts.q0.copy()
    for m, fib in enumerate(state.fibers):
        fib.X = parts.X[m].copy()
        fib.T = parts.T[m].copy()
    state.time += attempt
    _kinetics_and_contacts(state, attempt)     # replicated: same RNG streams on every rank
    if return_info:
        return state, dict(dt=attempt, iterations=iters, history=history, matvecs=op.matvecs)
    return state
