"""Implicit coupled stepping on the B200 (solver.py of the reference).

Same public API as /root/reference/pkg/src/slenderflow/solver.py --
GmresParams, StepLayout, BlockOperator, assemble_step_operator,
Preconditioner, gmres_solve, backward_euler_step, NonconvergenceError,
FactorizationError -- with the state, the Krylov basis and every block row
resident on the device.  One matvec is: fiber force densities and particle
wrenches from the candidate (sf_fiber_forces, sf_particle_wrenches), the HI
operator (sf_hi_apply), surface rows (subtracted double layer + rigid-body /
null-space terms, sf_surface_rows) and fiber rows (sf_fiber_rows).  The
Givens/Hessenberg bookkeeping of GMRES is a few dozen scalars per iteration
and stays on the host.
"""

import ctypes
import logging
import math
import os
import threading

import numpy as np

from . import _native, spectral
from .system import ConfigurationError, InteractionCache

LOG = logging.getLogger("paper_1602_05650_b200.solver")

BC_CODES = {"free": 0, "prescribedForceTorque": 1, "hingedToSurface": 2, "clampedToBody": 3}


class NonconvergenceError(RuntimeError):
    """GMRES ran out of iterations; carries the best iterate found (solver.py:40-47)."""

    def __init__(self, message, best=None, iterations=0, residuals=()):
        super().__init__(message)
        self.best = best
        self.iterations = iterations
        self.residuals = list(residuals)


class FactorizationError(RuntimeError):
    """A fiber self-block could not be inverted (solver.py:50-51)."""


class GmresParams:
    """Iteration controls (solver.py:54-64)."""

    def __init__(self, tolerance=1e-5, restart=60, max_iterations=500):
        if not 0.0 < tolerance < 1.0:
            raise ConfigurationError("GMRES tolerance must lie in (0, 1)")
        if restart < 1 or max_iterations < 1:
            raise ConfigurationError("restart length and iteration cap must be positive")
        self.tolerance = float(tolerance)
        self.restart = int(restart)
        self.max_iterations = int(max_iterations)


class StepLayout:
    """Index map of the stacked step unknowns (solver.py:67-110)."""

    def __init__(self, state):
        off = 0
        self.U, self.omega, self.q1 = [], [], []
        for part in state.particles:
            self.U.append(slice(off, off + 3))
            self.omega.append(slice(off + 3, off + 6))
            n = part.n_nodes
            self.q1.append(slice(off + 6, off + 6 + 3 * n))
            off += 6 + 3 * n
        self.q0 = None
        if state.periphery is not None:
            n0 = state.periphery.mesh.n_nodes
            self.q0 = slice(off, off + 3 * n0)
            off += 3 * n0
        self.fib_off = off
        self.X, self.T, self.fiber_block = [], [], []
        for fib in state.fibers:
            n = fib.n_nodes
            self.X.append(slice(off, off + 3 * n))
            self.T.append(slice(off + 3 * n, off + 4 * n))
            self.fiber_block.append(slice(off, off + 4 * n))
            off += 4 * n
        self.size = off

    def unpack(self, u):
        return _Parts([u[s] for s in self.U], [u[s] for s in self.omega],
                      [u[s].reshape(-1, 3) for s in self.q1],
                      u[self.q0].reshape(-1, 3) if self.q0 is not None else None,
                      [u[s].reshape(-1, 3) for s in self.X], [u[s] for s in self.T])


class _Parts:
    __slots__ = ("U", "omega", "q1", "q0", "X", "T")

    def __init__(self, U, omega, q1, q0, X, T):
        self.U, self.omega, self.q1, self.q0, self.X, self.T = U, omega, q1, q0, X, T


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _precision_mode(precision):
    """"fp64" (default) or "fp32c": the fiber x fiber pair sums in FP32
    arithmetic with FP64 accumulation (north_star variant, <= 1e-5 of FP64);
    every other term stays FP64."""
    from ._native import SF_MODE_FP32C, SF_MODE_FP64
    modes = {"fp64": SF_MODE_FP64, "fp32c": SF_MODE_FP32C}
    if precision not in modes:
        raise ConfigurationError(f"precision must be one of {sorted(modes)}")
    return modes[precision]


def _external_force_density_device(state, g, nb, n):
    """external_force_density (system.py:297-305) for one order class on the
    device, from the class's device tangents: the same elementwise sums in
    the same model order."""
    import torch
    f = torch.zeros((nb, n, 3), dtype=torch.float64, device=g.tang.device)
    for m in state.force_models:
        if m.kind == "uniformBodyForce":
            f += torch.as_tensor(m.f0 * m.direction, dtype=torch.float64, device=f.device)
        elif m.kind == "cytoplasmicPulling":
            f += (m.motor_force * m.motor_density) * g.tang
    return f


class _FiberBatch:
    """Fibers of one Chebyshev order: the frozen per-fiber operators and the
    sf_fiber_sys the per-fiber kernels take.  Unknown blocks and point ranges
    are addressed through per-fiber offset tables, so batches of different
    orders interleave freely in the reference's StepLayout."""

    def __init__(self, op, n, idx, g):
        import torch
        st = op.state
        dev = op.device
        f64 = dict(dtype=torch.float64, device=dev)
        nb = idx.size
        self.n, self.idx = n, idx
        fibs = [st.fibers[m] for m in idx]
        self.u_off = torch.as_tensor(np.array([op.layout.X[m].start for m in idx], dtype=np.int64),
                                     device=dev)
        self.pt_off = torch.as_tensor(op.cache.pt_off[idx].astype(np.int64), device=dev)
        self.Dpow = torch.empty((nb, 4, n, n), **f64)
        self.nodes = torch.tensor(spectral.grid(n - 1)[0], **f64)
        _native.call("sf_fiber_dpow", _ptr(g.D), _ptr(g.s_alpha), nb, n, _ptr(self.Dpow), _stream())
        self.K = torch.empty((nb, 3 * n, 3 * n), **f64)
        _native.call("sf_kdelta_build_batched", _ptr(g.X), _ptr(g.s), _ptr(g.s_alpha),
                     _ptr(g.tang), _ptr(g.wcc), nb, n, _ptr(g.delta),
                     1.0 / (8.0 * math.pi * op.mu), _ptr(self.K), _stream())
        eps = np.array([f.eps for f in fibs])
        self.E = torch.as_tensor(np.array([f.E for f in fibs], dtype=float), **f64)
        self.c_log = torch.as_tensor(-np.log(eps ** 2 * math.e) / (8.0 * math.pi * op.mu), **f64)
        self.Ldot = torch.as_tensor(np.array([f.Ldot for f in fibs], dtype=float), **f64)
        self.f_ext = None
        if st.force_models:
            self.f_ext = _external_force_density_device(st, g, nb, n)
        kinds = np.zeros((nb, 2), dtype=np.int32)
        par = np.zeros((nb, 2, 12))
        body = np.full(nb, -1, dtype=np.int32)
        for k, fib in enumerate(fibs):
            for e, bc in enumerate((fib.bc_plus, fib.bc_minus)):
                kinds[k, e] = BC_CODES[bc.kind]
                if bc.kind == "prescribedForceTorque":
                    par[k, e, 0:3] = bc.force
                    par[k, e, 3:6] = bc.torque
                elif bc.kind == "hingedToSurface":
                    par[k, e, 6:9] = bc.attachment
                    par[k, e, 9] = bc.stiffness
                elif bc.kind == "clampedToBody":
                    par[k, e, 10] = 0.0 if bc.tangent is None else 1.0
                    if e == 1:
                        body[k] = bc.body
        self.bc_kind = torch.as_tensor(kinds, device=dev)
        self.bc_par = torch.as_tensor(par, **f64)
        self.bc_body = torch.as_tensor(body, device=dev)
        self.geo = g
        self.sys = _native.FiberSys(
            nf=nb, n=n, D=_ptr(g.D), nodes=_ptr(self.nodes), Dpow=_ptr(self.Dpow), X=_ptr(g.X),
            tang=_ptr(g.tang), s_alpha=_ptr(g.s_alpha), L=_ptr(g.L), Ldot=_ptr(self.Ldot),
            E=_ptr(self.E), c_log=_ptr(self.c_log), c_two=2.0 / (8.0 * math.pi * op.mu),
            K=_ptr(self.K), f_ext=_ptr(self.f_ext), bc_kind=_ptr(self.bc_kind),
            bc_par=_ptr(self.bc_par), bc_body=_ptr(self.bc_body), np=op.np,
            pcenter=_ptr(op.pcenter), p_uoff=_ptr(op.p_uoff), fib_off=op.layout.fib_off,
            dt=op.dt, mu=op.mu, u_off=_ptr(self.u_off), pt_off=_ptr(self.pt_off))
        self.blocks = torch.empty((nb, 4 * n, 4 * n), **f64)
        _native.call("sf_fiber_self_blocks", ctypes.byref(self.sys), _ptr(self.blocks), _stream())


class BlockOperator:
    """Linear action of the implicit step system on the stacked unknowns,
    evaluated on the device (solver.py:187-364).  apply/rhs accept and return
    numpy arrays or CUDA tensors."""

    def __init__(self, state, dt, mu=None, backend=None, cache=None, implicit_coupling=True,
                 precision="fp64"):
        import torch
        if dt <= 0:
            raise ConfigurationError("time step must be positive")
        if not implicit_coupling:
            raise ConfigurationError("the device operator implements implicit coupling only")
        self.state = state
        self.dt = float(dt)
        self.mu = state.mu if mu is None else float(mu)
        if self.mu <= 0:
            raise ConfigurationError("viscosity must be positive")
        self.layout = StepLayout(state)
        self.cache = cache if cache is not None else \
            InteractionCache(state, backend=backend, mode=_precision_mode(precision))
        self.implicit_coupling = True
        self.device = self.cache.device
        dev = self.device
        f64 = dict(dtype=torch.float64, device=dev)
        c = self.cache
        nf = c.nf
        self.nf, self.n = nf, c.n_nodes
        np_ = len(state.particles)
        self.np = np_
        self.pcenter = self.cache.pcenter if np_ else None
        self.p_uoff = torch.as_tensor(np.array([s.start for s in self.layout.U], dtype=np.int64),
                                      device=dev) if np_ else None
        self.ext = (torch.as_tensor(np.stack([np.concatenate([p.F_ext, p.L_ext])
                                              for p in state.particles]), **f64) if np_ else None)
        # frozen fiber operators (refresh_geometry, fiber.py:133-147), one
        # uniform batch per Chebyshev order class
        self.batches = [_FiberBatch(self, n, idx, g) for n, idx, g in c.classes if idx.size]
        if len(self.batches) == 1:
            b = self.batches[0]
            self.sys, self.Dpow, self.K = b.sys, b.Dpow, b.K
            self.fiber_blocks = b.blocks
        else:
            self.sys = None
            blocks = [None] * nf
            for b in self.batches:
                for k, m in enumerate(b.idx):
                    blocks[m] = b.blocks[k]
            self.fiber_blocks = blocks
        # surface data per particle / periphery, the cache's device arrays
        self.surf = []
        for i, part in enumerate(state.particles):
            m = c.surfaces[i][0]
            nodes, nrm, w = c.surface_arrays[i]
            self.surf.append(dict(kind=0, pi=i, nodes=nodes, nrm=nrm, w=w, n=m.n_nodes, area=m.area,
                                  center=self.pcenter[i], sl=self.layout.q1[i],
                                  uom=self.layout.U[i].start, tsl=c.particle_slices[i]))
        if state.periphery is not None:
            m = c.surfaces[-1][0]
            nodes, nrm, w = c.surface_arrays[-1]
            self.surf.append(dict(kind=1, nodes=nodes, nrm=nrm, w=w, n=m.n_nodes, area=m.area,
                                  center=None, sl=self.layout.q0, uom=None,
                                  tsl=c.periphery_slice))
        # scratch
        self._f = torch.empty((int(c.node_counts.sum()), 3), **f64)
        self._wf = torch.empty((max(nf, 1), 6), **f64)
        self._wr = torch.empty((max(np_, 1), 6), **f64)
        self._wr_k = torch.empty((max(np_, 1), 6), **f64) if len(self.batches) > 1 else None
        self._ubar = torch.empty((c.n_targets, 3), **f64)
        self._work = torch.empty(16, **f64)
        self._pcache = None
        self.matvecs = 0

    @property
    def shape(self):
        return (self.layout.size, self.layout.size)

    # ------------------------------------------------------------- rows
    def _densities(self, u):
        """Surface densities in the cache's surface order (particles, periphery)."""
        import torch
        if not self.surf:
            return None
        return torch.cat([u[s["sl"]] for s in self.surf]).reshape(-1, 3)

    def rows_device(self, u, constants, out=None):
        import torch
        c = self.cache
        st = _stream()
        if out is None:
            out = torch.empty_like(u)
        for b in self.batches:
            _native.call("sf_fiber_forces", ctypes.byref(b.sys), _ptr(u), int(constants),
                         _ptr(self._f), st)
        if self.np:
            if not self.batches:
                self._wr.zero_()
                if constants:
                    self._wr[:self.np].copy_(self.ext)
            for k, b in enumerate(self.batches):     # classes summed in a fixed order
                _native.call("sf_particle_wrenches", ctypes.byref(b.sys), _ptr(u),
                             _ptr(self.ext) if k == 0 else None, int(constants), _ptr(self._wf),
                             _ptr(self._wr if k == 0 else self._wr_k), st)
                if k:
                    self._wr.add_(self._wr_k)
        q = self._densities(u)
        # the skipped-pair counts depend only on the frozen geometry (which
        # pairs are cross-group and closer than 1e-12), not on u: check them
        # on the cache's first application and never sync on them again
        check = not getattr(c, "_bad_checked", False)
        ubar = c.apply(self._f, q, self._wr[:self.np] if self.np else None, out=self._ubar,
                       check=check)
        c._bad_checked = True
        pref_dl = -3.0 / (4.0 * math.pi * self.mu)
        for s in self.surf:
            qs = u[s["sl"]]
            rows = out[s["sl"]]
            _native.call("sf_stresslet_sum_subtracted", _ptr(s["nodes"]), _ptr(s["nrm"]),
                         _ptr(s["w"]), _ptr(qs), s["n"], pref_dl, _ptr(rows), st)
            ub = ubar[s["tsl"]]
            if s["kind"] == 0:
                _native.call("sf_wrench_flow", _ptr(s["nodes"]), s["n"], _ptr(s["center"]),
                             _ptr(self._wr[s["pi"]]), self.mu, _ptr(rows), st)
                uom = u[s["uom"]:s["uom"] + 6]
                _native.call("sf_surface_rows", 0, _ptr(s["nodes"]), _ptr(s["nrm"]), _ptr(s["w"]),
                             s["n"], _ptr(s["center"]), s["area"], _ptr(qs), _ptr(ub), _ptr(uom),
                             self.mu, _ptr(self._work), _ptr(rows),
                             _ptr(out[s["uom"]:s["uom"] + 6]), st)
            else:
                _native.call("sf_surface_rows", 1, _ptr(s["nodes"]), _ptr(s["nrm"]), _ptr(s["w"]),
                             s["n"], None, s["area"], _ptr(qs), _ptr(ub), None, self.mu,
                             _ptr(self._work), _ptr(rows), None, st)
        for b in self.batches:
            _native.call("sf_fiber_rows", ctypes.byref(b.sys), _ptr(u), _ptr(self._f),
                         _ptr(ubar[c.fiber_slice]), int(constants), _ptr(out), st)
        self.matvecs += 1
        return out

    def fiber_rows_local_device(self, u, out):
        """Fiber rows of A u without the complementary velocity (ubar = 0):
        each fiber's self terms, elastic operators and boundary rows,
        including the clamped ends' dependence on the particle's U, omega.
        Writes the fiber entries of out."""
        import torch
        c = self.cache
        npts = c.fiber_slice.stop - c.fiber_slice.start
        if getattr(self, "_zero_ubar", None) is None or self._zero_ubar.shape[0] != npts:
            self._zero_ubar = torch.zeros((max(npts, 1), 3), dtype=torch.float64,
                                          device=self.device)
        for b in self.batches:
            _native.call("sf_fiber_rows", ctypes.byref(b.sys), _ptr(u), None, _ptr(self._zero_ubar),
                         0, _ptr(out), _stream())
        return out

    def particle_rows_device(self, u, out=None):
        """Rows of the particle blocks [U omega q1 per particle] driven by the
        FIBER unknowns of u alone (its surface entries are ignored): the
        fibers' attachment wrenches, their wrench flow and the fibers'
        velocity at the particle nodes (pair sums, near corrections,
        completion flows).  This is A[particle rows, fiber columns] @ u, the
        coupling block of the body-coupled preconditioner; it evaluates only
        the particle targets (a target-ranged InteractionCache), not the
        fiber x fiber sum."""
        import torch
        st = _stream()
        pend = self.layout.q1[-1].stop
        if out is None:     # a reused buffer: callers consume it before the next call
            if getattr(self, "_prow", None) is None:
                self._prow = torch.empty(pend, dtype=torch.float64, device=self.device)
            out = self._prow
        if self._pcache is None:
            npn = sum(s["n"] for s in self.surf if s["kind"] == 0)
            self._pcache = InteractionCache(self.state, mode=self.cache.mode,
                                            target_range=(0, npn))
            nss = sum(s["n"] for s in self.surf)
            self._pzero_q = torch.zeros((max(nss, 1), 3), dtype=torch.float64, device=self.device)
            self._pzero_u = torch.zeros(6, dtype=torch.float64, device=self.device)
            self._pubar = torch.empty((npn, 3), dtype=torch.float64, device=self.device)
        pc = self._pcache
        for b in self.batches:
            _native.call("sf_fiber_forces", ctypes.byref(b.sys), _ptr(u), 0, _ptr(self._f), st)
        for k, b in enumerate(self.batches):
            _native.call("sf_particle_wrenches", ctypes.byref(b.sys), _ptr(u), None, 0,
                         _ptr(self._wf), _ptr(self._wr if k == 0 else self._wr_k), st)
            if k:
                self._wr.add_(self._wr_k)
        q = self._pzero_q[:sum(s["n"] for s in self.surf)] if self.surf else None
        ubar = pc.apply(self._f, q, self._wr[:self.np], out=self._pubar, check=False)
        out.zero_()
        for s in self.surf:
            if s["kind"] != 0:
                continue
            rows = out[s["sl"]]
            _native.call("sf_wrench_flow", _ptr(s["nodes"]), s["n"], _ptr(s["center"]),
                         _ptr(self._wr[s["pi"]]), self.mu, _ptr(rows), st)
            _native.call("sf_surface_rows", 0, _ptr(s["nodes"]), _ptr(s["nrm"]), _ptr(s["w"]),
                         s["n"], _ptr(s["center"]), s["area"], _ptr(self._pzero_q[:s["n"]]),
                         _ptr(ubar[pc.particle_slices[s["pi"]]]), _ptr(self._pzero_u), self.mu,
                         _ptr(self._work), _ptr(rows), _ptr(out[s["uom"]:s["uom"] + 6]), st)
        return out

    def particle_block_matrix(self):
        """Dense A[particle rows, particle columns] (own-particle terms; the
        particles' mutual coupling through the fluid is left out), assembled
        on the device from the row definitions (solver.py:332-346):
        U - <q>/mu, omega - <arm x q>/mu, and the on-surface double layer of
        q1 (body.second_kind_matrix without the jump) - (U + omega x arm)."""
        import torch
        pend = self.layout.q1[-1].stop
        f64 = dict(dtype=torch.float64, device=self.device)
        B = torch.zeros((pend, pend), **f64)
        eye = torch.eye(3, **f64)
        for s in self.surf:
            if s["kind"] != 0:
                continue
            a, n = s["uom"], s["n"]
            q0 = a + 6
            arm = s["nodes"] - s["center"]
            cross = torch.zeros((n, 3, 3), **f64)          # [arm]_x v = arm x v
            cross[:, 0, 1], cross[:, 0, 2] = -arm[:, 2], arm[:, 1]
            cross[:, 1, 0], cross[:, 1, 2] = arm[:, 2], -arm[:, 0]
            cross[:, 2, 0], cross[:, 2, 1] = -arm[:, 1], arm[:, 0]
            wj = s["w"] / (s["area"] * self.mu)
            B[a:a + 3, a:a + 3] = eye
            B[a + 3:a + 6, a + 3:a + 6] = eye
            B[a:a + 3, q0:q0 + 3 * n] = -(wj[:, None, None] * eye).permute(1, 0, 2).reshape(3, 3 * n)
            B[a + 3:a + 6, q0:q0 + 3 * n] = -(wj[:, None, None] * cross).permute(1, 0, 2).reshape(
                3, 3 * n)
            B[q0:q0 + 3 * n, a:a + 3] = -eye.repeat(n, 1)
            B[q0:q0 + 3 * n, a + 3:a + 6] = cross.reshape(3 * n, 3)
            B[q0:q0 + 3 * n, q0:q0 + 3 * n] = _double_layer_matrix(s["nodes"], s["nrm"], s["w"],
                                                                   self.mu)
        return B

    def _to_dev(self, u):
        import torch
        return torch.as_tensor(u, dtype=torch.float64, device=self.device).contiguous()

    def apply(self, u):
        """A @ u, strictly linear (solver.py:217-222)."""
        is_np = isinstance(u, np.ndarray)
        if u.shape != (self.layout.size,):
            raise ValueError(f"expected a vector of length {self.layout.size}")
        out = self.rows_device(self._to_dev(u), False)
        return out.cpu().numpy() if is_np else out

    def rhs_device(self):
        import torch
        zero = torch.zeros(self.layout.size, dtype=torch.float64, device=self.device)
        return -self.rows_device(zero, True)

    def rhs(self):
        """Right-hand side of every candidate-independent term (solver.py:224-227)."""
        return self.rhs_device().cpu().numpy()

    def materialize(self):
        n = self.layout.size
        A = np.empty((n, n))
        e = np.zeros(n)
        for j in range(n):
            e[j] = 1.0
            A[:, j] = self.apply(e)
            e[j] = 0.0
        return A


def _double_layer_matrix(x, n, w, mu):
    """Dense matrix of double_layer_onsurface (body.py:254-262: the
    subtracted stresslet sum, kernels.py:216-249): off-diagonal 3x3 blocks
    pref w_j (n_j . r) r r^T / r^5, diagonal blocks minus their row sums
    (body.second_kind_matrix with interior=False)."""
    import torch
    N = x.shape[0]
    pref = -3.0 / (4.0 * math.pi * mu)
    r = x[:, None, :] - x[None, :, :]
    d2 = (r * r).sum(dim=2)
    d2.fill_diagonal_(1.0)
    scal = pref * (r * n[None, :, :]).sum(dim=2) / (d2 * d2 * torch.sqrt(d2)) * w[None, :]
    idx = torch.arange(N, device=x.device)
    scal[idx, idx] = 0.0
    blocks = scal[:, :, None, None] * r[:, :, :, None] * r[:, :, None, :]
    rowsum = blocks.sum(dim=1)
    blocks[idx, idx] = -rowsum
    return blocks.permute(0, 2, 1, 3).reshape(3 * N, 3 * N)


def assemble_step_operator(state, dt, mu=None, backend=None, cache=None, implicit_coupling=True,
                           precision="fp64"):
    op = BlockOperator(state, dt, mu=mu, backend=backend, cache=cache,
                       implicit_coupling=implicit_coupling, precision=precision)
    return op, op.rhs_device()


_PARTICLE_INV_CACHE = []      # [(key arrays, mu, device, inverse)], most recent first
_PARTICLE_INV_LOCK = threading.Lock()   # emulated ranks (dsolver.ThreadComm) share it


def _particle_block_inverse(op):
    """A_pp^-1 (BlockOperator.particle_block_matrix, own-particle blocks) as
    an explicit matrix: one GEMV per preconditioner apply (a single-RHS
    library triangular solve of this size measured ~0.8 ms, the GEMV ~20 us).
    A_pp depends only on each particle's nodes relative to its centre,
    normals and weights, so the inverse is reused while the particles
    translate (relative geometry equal to 1e-13 of its size)."""
    import torch
    key = [(s["nodes"] - s["center"], s["nrm"], s["w"]) for s in op.surf if s["kind"] == 0]

    def same(a, b):
        """Relative geometry equal to 1e-13 (one flag read on the device)."""
        if len(a) != len(b):
            return False
        flags = []
        for (r1, n1, w1), (r2, n2, w2) in zip(a, b):
            if r1.shape != r2.shape or r1.device != r2.device:
                return False
            scale = torch.clamp(r1.abs().max(), min=1.0)
            flags.append(((r1 - r2).abs().max() <= 1e-13 * scale) & ((n1 - n2).abs().max() <= 1e-13)
                         & ((w1 - w2).abs().max() <= 1e-13 * w1.abs().max()))
        return bool(torch.stack(flags).all())
    with _PARTICLE_INV_LOCK:
        for idx, entry in enumerate(_PARTICLE_INV_CACHE):
            k, mu, dev, inv = entry
            if mu == op.mu and dev == op.device and same(k, key):
                del _PARTICLE_INV_CACHE[idx]          # by position: entries hold tensors
                _PARTICLE_INV_CACHE.insert(0, entry)
                return inv
    A = op.particle_block_matrix()
    if not bool(torch.isfinite(A).all()):
        raise FactorizationError("particle block is not finite")
    inv, info = torch.linalg.inv_ex(A)
    if int(info.item()) != 0 or not bool(torch.isfinite(inv).all()):
        raise FactorizationError("particle block is singular")
    with _PARTICLE_INV_LOCK:
        _PARTICLE_INV_CACHE.insert(0, (key, op.mu, op.device, inv))
        del _PARTICLE_INV_CACHE[4:]
    return inv


class Preconditioner:
    """Block Jacobi: equilibrated exact fiber-block inverses, diagonal on
    surface rows (solver.py:375-429), factored and applied on the device
    (one batch of block factors per Chebyshev order class).

    body_coupling=True (not in the reference; off by default) additionally
    inverts, exactly, the rigid particles' own blocks [U omega q1] together
    with their coupling to the fibers: the particle rows' dependence on every
    fiber unknown (attachment wrenches, wrench flow, fiber velocity at the
    particle nodes) and the fiber rows' dependence on U and omega (clamped
    ends).  Only the fiber <-> fiber and periphery couplings stay outside.
    Solved by a Schur complement on the particle unknowns:
        W = D^-1 A[f, U omega],  S = A[p, p] - A[p, f] W,
        z_p = S^-1 (v_p - A[p, f] D^-1 v_f),  z_f = D^-1 v_f - W z_(U omega).
    S^-1 by Sherman-Morrison-Woodbury around A[p, p]^-1 (S differs from it
    in the 6 U/omega columns per particle; A[p, p] is translation invariant,
    so its inverse is cached across steps; S^-1 is then a rank-6 update of
    it).  Per apply: the block solves, one particle-rows evaluation
    (BlockOperator.particle_rows_device) and one GEMV with S^-1.  It
    targets asters, where GMRES with block Jacobi needs 175 (C2) to 480 (C4)
    iterations; the solution is the same to the GMRES tolerance."""

    def __init__(self, op, body_coupling=False):
        import torch
        self.layout = op.layout
        self.device = op.device
        f64 = dict(dtype=torch.float64, device=op.device)
        self.off0 = op.layout.fib_off
        st = _stream()
        self.factors = []       # (LU, r, c, piv, nb, m, u_off) per batch
        for b in op.batches:
            nb, m = b.idx.size, 4 * b.n
            A = b.blocks.clone()
            if not bool(torch.isfinite(A).all()):
                raise FactorizationError("fiber self-block is not finite")
            if m <= 256:
                # shared-memory LU for m <= 160, blocked global-memory LU up to 256
                r = torch.empty((nb, m), **f64)
                c = torch.empty((nb, m), **f64)
                piv = torch.empty((nb, m), dtype=torch.int32, device=op.device)
                info = torch.empty(nb, dtype=torch.int32, device=op.device)
                _native.call("sf_block_lu", _ptr(A), nb, m, _ptr(r), _ptr(c), _ptr(piv),
                             _ptr(info), st)
                LU = A
            else:
                # larger blocks: equilibrate on the device and factor with the
                # batched library getrf (outside every BASELINE config)
                r = A.abs().amax(dim=2)
                if bool((r == 0).any()):
                    raise FactorizationError("fiber self-block is singular")
                A = A / r[:, :, None]
                c = A.abs().amax(dim=1)
                A = A / c[:, None, :]
                LUt, pv, inf = torch.linalg.lu_factor_ex(A)
                info = torch.where(inf != 0, 3, 0).to(torch.int32)
                LU = LUt.transpose(1, 2).contiguous()
                piv = (pv - 1).to(torch.int32).contiguous()
            bad = info.cpu().numpy()
            if np.any(bad == 1):
                raise FactorizationError(
                    f"fiber {int(b.idx[np.argmax(bad == 1)])} self-block is not finite")
            if np.any(bad == 2) or np.any(bad == 3):
                raise FactorizationError(
                    f"fiber {int(b.idx[np.argmax(bad > 1)])} self-block is singular")
            self.factors.append((LU, r, c, piv, nb, m, b.u_off))
        uniform = len(self.factors) == 1 and bool(
            (self.factors[0][6] == self.off0 + 4 * op.batches[0].n
             * torch.arange(op.nf, device=op.device)).all()) if op.nf else True
        self.uniform = uniform
        if len(self.factors) == 1:
            self.LU, self.r, self.c, self.piv, self.nb, self.m = self.factors[0][:6]
        diag = torch.ones(self.off0, **f64)
        pref = -3.0 / (4.0 * math.pi * op.mu)
        for s in op.surf:
            rs = torch.empty((s["n"], 3, 3), **f64)
            _native.call("sf_stresslet_rowsum", _ptr(s["nodes"]), _ptr(s["nrm"]), _ptr(s["w"]),
                         s["n"], pref, _ptr(rs), st)
            d = -torch.diagonal(rs, dim1=1, dim2=2)
            if s["kind"] == 1:
                d = d + 1.0 / op.mu
                d = d + (s["nrm"] ** 2) * s["w"][:, None] / (op.mu * s["area"])
            diag[s["sl"]] = d.reshape(-1)
        if bool((diag == 0).any()):
            raise FactorizationError("zero diagonal entry in a surface block")
        self.diag = diag
        self.coupled = None
        if body_coupling and op.np and op.nf:
            self._setup_body_coupling(op)

    def _setup_body_coupling(self, op):
        import torch
        lay = op.layout
        n, fo = lay.size, lay.fib_off
        pend = lay.q1[-1].stop
        f64 = dict(dtype=torch.float64, device=self.device)
        cols = [k for i in range(op.np) for k in range(lay.U[i].start, lay.U[i].start + 6)]
        e = torch.zeros(n, **f64)
        W = torch.empty((n - fo, len(cols)), **f64)
        v = torch.zeros(n, **f64)
        for k, j in enumerate(cols):
            # fiber rows of the U / omega columns: only the clamped ends see
            # them, and U, omega are no flow sources, so ubar = 0 is exact
            e[j] = 1.0
            op.fiber_rows_local_device(e, v)
            e[j] = 0.0
            W[:, k] = self._block_jacobi(v)[fo:]
        # S = A_pp - Z E^T with Z = A_pf W and E the U/omega columns, inverted
        # by Sherman-Morrison-Woodbury around A_pp^-1, which depends only on
        # the particles' geometry relative to their centres (translation
        # invariant), so it is computed once and reused while they translate
        Ainv = _particle_block_inverse(op)
        t = torch.zeros(n, **f64)
        Z = torch.empty((pend, len(cols)), **f64)
        for k in range(len(cols)):
            t[fo:] = W[:, k]
            Z[:, k] = op.particle_rows_device(t)
        colt = torch.as_tensor(cols, device=self.device)
        AZ = Ainv @ Z
        C = torch.eye(len(cols), **f64) - AZ[colt]
        Cinv, info = torch.linalg.inv_ex(C)
        if int(info.item()) != 0 or not bool(torch.isfinite(Cinv).all()) or \
                not bool(torch.isfinite(AZ).all()):
            raise FactorizationError("particle Schur complement is singular")
        Sinv = torch.addmm(Ainv, AZ, Cinv @ Ainv[colt])      # rank-6np update
        contiguous = cols == list(range(cols[0], cols[0] + len(cols)))
        self.coupled = dict(op=op, pend=pend, fo=fo, W=W, Sinv=Sinv, cols=colt,
                            cslice=slice(cols[0], cols[0] + len(cols)) if contiguous else None)

    def apply_device(self, v, out=None):
        out = self._block_jacobi(v, out)
        cp = self.coupled
        if cp is not None:
            import torch
            pend, fo = cp["pend"], cp["fo"]
            r = torch.sub(v[:pend], cp["op"].particle_rows_device(out))
            zb = torch.mv(cp["Sinv"], r, out=out[:pend])
            zc = zb[cp["cols"]] if cp["cslice"] is None else zb[cp["cslice"]]
            out[fo:].addmv_(cp["W"], zc, alpha=-1.0)
        return out

    def _block_jacobi(self, v, out=None):
        import torch
        if out is None:
            out = torch.empty_like(v)
        st = _stream()
        if self.uniform and len(self.factors) == 1:
            LU, r, c, piv, nb, m, _ = self.factors[0]
            _native.call("sf_precond_apply", _ptr(LU), _ptr(r), _ptr(c), _ptr(piv), nb, m,
                         self.off0, _ptr(self.diag), self.off0, _ptr(v), _ptr(out), st)
            return out
        _native.call("sf_precond_apply", None, None, None, None, 0, 0, self.off0, _ptr(self.diag),
                     self.off0, _ptr(v), _ptr(out), st)
        for LU, r, c, piv, nb, m, uoff in self.factors:
            _native.call("sf_block_solve", _ptr(LU), _ptr(r), _ptr(c), _ptr(piv), nb, m,
                         _ptr(uoff), _ptr(v), _ptr(out), st)
        return out

    def apply(self, v):
        import torch
        if isinstance(v, np.ndarray):
            return self.apply_device(torch.as_tensor(v, device=self.device)).cpu().numpy()
        return self.apply_device(v.contiguous())


class _DeviceVectors:
    """Deterministic dot / axpy helpers on device vectors (sf_dot etc.)."""

    def __init__(self, device):
        import torch
        self.work = torch.empty(4 * 296, dtype=torch.float64, device=device)

    def dot_into(self, x, y, out, sqrt_mode=False):
        _native.call("sf_dot", _ptr(x), _ptr(y), x.numel(), _ptr(self.work), _ptr(out),
                     int(sqrt_mode), _stream())


def _as_apply(obj, device):
    import torch
    if obj is None:
        return lambda v: v
    if hasattr(obj, "apply_device"):
        return obj.apply_device
    if hasattr(obj, "rows_device"):
        return lambda v: obj.rows_device(v, False)
    if hasattr(obj, "apply"):
        fn = obj.apply
    elif isinstance(obj, np.ndarray):
        M = torch.as_tensor(obj, dtype=torch.float64, device=device)
        return lambda v: M @ v
    elif callable(obj):
        fn = obj
    else:
        raise TypeError("operator must expose .apply, be a matrix, or be callable")

    def wrapped(v):
        r = fn(v)
        return torch.as_tensor(r, dtype=torch.float64, device=device)
    return wrapped


_GMRES_STATUS_RING = 8


def _status_lag(operator):
    """Arnoldi steps queued ahead of the convergence read.  With lag 1 the
    host enqueues step k+1 before it waits for step k's status, so the GPU
    never idles on the host; the price is one speculative matvec when the
    solve converges, which only pays off while a matvec is cheap next to
    the host's per-step launch work.  SF_GMRES_LAG overrides."""
    env = os.environ.get("SF_GMRES_LAG")
    if env is not None:
        return max(0, int(env))
    cache = getattr(operator, "cache", None)
    pairs = getattr(cache, "pairs_per_apply", None) if cache is not None else None
    if pairs is None:
        return 1
    return 1 if pairs < 2e10 else 0


def gmres_solve(operator, preconditioner, rhs, params=None, x0=None, lag=None):
    """Left-preconditioned restarted GMRES (solver.py:444-516), entirely on
    the device: Krylov basis, fused modified Gram-Schmidt (sf_gmres_mgs),
    Hessenberg rotations, residual estimate and the restart update
    (sf_gmres_givens / sf_gmres_update).  Per Arnoldi step the host reads one
    4-double status record, copied asynchronously into pinned memory and
    consumed `lag` steps late (see _status_lag); once per cycle it reads the
    scalars and the residual history.  Returns (solution, iterations,
    residual history); the solution has the type of `rhs` (numpy or CUDA
    tensor)."""
    import torch
    if params is None:
        params = GmresParams()
    host_io = isinstance(rhs, np.ndarray)
    device = getattr(operator, "device", None) or torch.device("cuda")
    rhs_d = torch.as_tensor(rhs, dtype=torch.float64, device=device).contiguous()
    apply_a = _as_apply(operator, device)
    apply_m = _as_apply(preconditioner, device)
    vec = _DeviceVectors(device)
    st = _stream()
    n = rhs_d.numel()
    fused = os.environ.get("SF_GMRES_FUSED", "1") != "0"
    if lag is None:
        lag = _status_lag(operator)

    def ret(x):
        return x.cpu().numpy() if host_io else x

    scal = torch.empty(2, dtype=torch.float64, device=device)
    b = apply_m(rhs_d)
    vec.dot_into(b, b, scal[0:1], sqrt_mode=True)
    beta0 = float(scal[0].item())
    if beta0 == 0.0:
        return ret(torch.zeros(n, dtype=torch.float64, device=device)), 0, [0.0]
    warm = x0 is not None
    x = (torch.as_tensor(x0, dtype=torch.float64, device=device).clone() if warm
         else torch.zeros(n, dtype=torch.float64, device=device))
    R, maxit = params.restart, params.max_iterations
    V = torch.empty((R + 1, n), dtype=torch.float64, device=device)
    hcol = torch.empty(R + 2, dtype=torch.float64, device=device)
    lib = _native.load(require_device=True)
    ns = int(lib.sf_gmres_state_doubles(R, maxit))
    gs = torch.zeros(ns, dtype=torch.float64, device=device)
    status = torch.zeros(4, dtype=torch.float64, device=device)
    ring = torch.zeros((_GMRES_STATUS_RING, 4), dtype=torch.float64).pin_memory()
    events = [torch.cuda.Event() for _ in range(_GMRES_STATUS_RING)]
    hist_off = ns - maxit
    _native.call("sf_gmres_reset", _ptr(gs), R, maxit, beta0, params.tolerance, st)
    history = []
    iters = 0
    # SF_GMRES_GRAPH=1: one Arnoldi step (matvec, preconditioner, fused MGS,
    # Givens) captured once as a CUDA graph and replayed for every later
    # step; the step index is read from the device state, so the same graph
    # serves every k (_graph_wanted).  Device-native operators only.
    graph = _ArnoldiGraph.create(operator, preconditioner, V, hcol, gs, hist_off - 8, R, vec,
                                 fused) if n else None
    while True:
        r = b - apply_m(apply_a(x)) if (iters or warm) else b
        vec.dot_into(r, r, scal[0:1], sqrt_mode=True)
        beta = float(scal[0].item())
        if beta / beta0 <= params.tolerance:
            return ret(x), iters, history or [beta / beta0]
        _native.call("sf_gmres_cycle", _ptr(gs), R, _ptr(scal[0:1]), _ptr(r), _ptr(V[0]), n, st)
        k = 0
        pending = []
        while k < R and iters + k < maxit:
            if graph is not None and graph.ready(iters + k):
                graph.step(V[k], status)
            else:
                _eager_arnoldi_step(apply_a, apply_m, V, k, hcol, gs, R, vec, fused, n, status)
            slot = k % _GMRES_STATUS_RING
            ring[slot].copy_(status, non_blocking=True)
            events[slot].record()
            pending.append(slot)
            k += 1
            done = False
            while len(pending) > lag:
                s0 = pending.pop(0)
                events[s0].synchronize()
                if ring[s0, 0] != 0.0:
                    done = True
                    break
            if done:
                break
        _native.call("sf_gmres_update", _ptr(V), n, _ptr(gs), R, _ptr(x), n, st)
        sc = gs[hist_off - 8:].cpu().numpy()            # scalars + history (one read per cycle)
        new_iters = int(sc[1])
        history.extend(float(h) for h in sc[8 + iters:8 + new_iters])
        iters = new_iters
        rel = history[-1] if history else 0.0
        if rel <= params.tolerance:
            return ret(x), iters, history
        if iters >= maxit:
            raise NonconvergenceError(
                f"GMRES did not reach {params.tolerance:g} within "
                f"{params.max_iterations} iterations (residual {rel:.3e})",
                best=ret(x), iterations=iters, residuals=history)


def _eager_arnoldi_step(apply_a, apply_m, V, k, hcol, gs, R, vec, fused, n, status):
    """One Arnoldi step launched kernel by kernel (solver.py:482-505)."""
    st = _stream()
    w = apply_m(apply_a(V[k])).contiguous()
    if fused:
        # wnorm, modified Gram-Schmidt, |w| and V[k+1] = w/|w| in one launch
        _native.call("sf_gmres_mgs", _ptr(V), n, k, _ptr(w), n, _ptr(hcol), R, _ptr(vec.work), st)
    else:
        vec.dot_into(w, w, hcol[R + 1:R + 2], sqrt_mode=True)   # wnorm
        for j in range(k + 1):                                   # modified Gram-Schmidt
            vec.dot_into(V[j], w, hcol[j:j + 1])
            _native.call("sf_axpy_dev", _ptr(hcol[j:j + 1]), -1.0, 0, _ptr(V[j]), _ptr(w), n, st)
        vec.dot_into(w, w, hcol[k + 1:k + 2], sqrt_mode=True)
        _native.call("sf_axpy_dev", _ptr(hcol[k + 1:k + 2]), 1.0, 2, _ptr(w), _ptr(V[k + 1]), n, st)
    _native.call("sf_gmres_givens", _ptr(hcol), _ptr(gs), R, k, _ptr(status), st)


# Replaying the captured Arnoldi step removes the launch bubbles between the
# ~40 kernels of a step: at C2 the steady step period drops from 2.03 to
# 1.99 ms (tools/step_timeline.py), but whole C2 steps measured 377-400 ms
# against 381 ms eager (tools/c2_step_ab.py: per-solve capture and replay
# variance), and at C1 the ~1-2 ms capture per solve outweighs it (6.5-7.2
# vs 5.5 ms per step).  Opt-in: SF_GMRES_GRAPH=1.
def _graph_wanted(operator):
    return os.environ.get("SF_GMRES_GRAPH", "0") == "1"


class _ArnoldiGraph:
    """The Arnoldi step of gmres_solve as one CUDA graph: A vin -> tmp,
    M tmp -> w (both into fixed buffers), the fused MGS and the Givens
    update with the step index read from the device (sf_gmres_mgs_dk,
    sf_gmres_givens with k = -1).  Captured after the first eagerly run step
    (so every workspace, side stream and lazily built buffer exists) and
    replayed for the rest of the solve; the launch work per step drops from
    ~30 host-side kernel launches to one graph launch.  Falls back to the
    eager path if the capture fails."""

    @classmethod
    def create(cls, operator, preconditioner, V, hcol, gs, sc_off, R, vec, fused):
        if not fused or not _graph_wanted(operator):
            return None
        if not hasattr(operator, "rows_device"):
            return None
        if preconditioner is not None and not hasattr(preconditioner, "apply_device"):
            return None
        return cls(operator, preconditioner, V, hcol, gs, sc_off, R, vec)

    def __init__(self, operator, preconditioner, V, hcol, gs, sc_off, R, vec):
        import torch
        self.op, self.prec = operator, preconditioner
        self.V, self.hcol, self.gs, self.R, self.vec = V, hcol, gs, R, vec
        self.sc = gs[sc_off:]
        n = V.shape[1]
        self.vin = torch.empty(n, dtype=torch.float64, device=V.device)
        self.tmp = torch.empty_like(self.vin)
        self.w = torch.empty_like(self.vin)
        self.status = torch.empty(4, dtype=torch.float64, device=V.device)
        # the library keys its scratch and side streams by stream: the step
        # is warmed up and captured on one dedicated stream, so the graph
        # holds that stream's (already grown) workspaces
        self.stream = torch.cuda.Stream(device=V.device)
        self.graph = None
        self.warm = False
        self.failed = False

    def ready(self, step):
        """Step 0 runs eagerly on the caller's stream, step 1 eagerly on the
        capture stream (warm-up), step 2 is captured, later steps replay."""
        return step >= 1 and not self.failed

    def _body(self):
        st = _stream()
        self.op.rows_device(self.vin, False, self.tmp)
        if self.prec is None:
            self.w.copy_(self.tmp)
        else:
            self.prec.apply_device(self.tmp, self.w)
        n = self.V.shape[1]
        _native.call("sf_gmres_mgs_dk", _ptr(self.V), n, _ptr(self.sc), _ptr(self.w), n,
                     _ptr(self.hcol), self.R, _ptr(self.vec.work), st)
        _native.call("sf_gmres_givens", _ptr(self.hcol), _ptr(self.gs), self.R, -1,
                     _ptr(self.status), st)

    def step(self, vk, status):
        import torch
        self.vin.copy_(vk)
        cur = torch.cuda.current_stream()
        if not self.warm:
            self.stream.wait_stream(cur)
            with torch.cuda.stream(self.stream):
                self._body()
            cur.wait_stream(self.stream)
            self.warm = True
            status.copy_(self.status)
            return
        if self.graph is None:
            g = torch.cuda.CUDAGraph()
            matvecs = getattr(self.op, "matvecs", None)
            try:
                # capture_begin/end directly: torch.cuda.graph() would also run
                # gc.collect() and empty_cache() on every solve (measured
                # +140 ms per C2 step in a process holding a C5 state)
                self.stream.wait_stream(cur)
                with torch.cuda.stream(self.stream):
                    g.capture_begin(capture_error_mode=os.environ.get(
                        "SF_GMRES_CAPTURE_MODE", "thread_local"))
                    try:
                        self._body()
                    finally:
                        g.capture_end()
            except Exception as err:      # noqa: BLE001 - capture unsupported: stay eager
                LOG.warning("GMRES step graph capture failed (%s); running eagerly", err,
                            exc_info=os.environ.get("SF_GMRES_CAPTURE_TRACE") == "1")
                self.failed = True
                torch.cuda.synchronize()
                if matvecs is not None:
                    self.op.matvecs = matvecs
                self._body()
                status.copy_(self.status)
                return
            if matvecs is not None:
                self.op.matvecs = matvecs
            self.graph = g
        self.graph.replay()
        if hasattr(self.op, "matvecs"):
            self.op.matvecs += 1
        status.copy_(self.status)


def _kinetics_and_contacts(state, dt):
    """Polymerization kinetics and contact models after the geometry update
    (solver.py:574-588): per-fiber scalar host logic with the reference's
    RNG draws, run by the reference's own functions (_reference.py) on these
    host objects; the resulting Ldot enters the next step's device rows."""
    from . import _reference
    ref_fiber = _reference.module("fiber")
    ref_system = _reference.module("system")
    for fib in state.fibers:
        if fib.growth_state == ref_fiber.STALLED:
            continue
        load = np.zeros(3)
        if fib.bc_plus.kind == "hingedToSurface":
            load = fib.bc_plus.stiffness * (fib.X[0] - fib.bc_plus.attachment)
        kin = fib.kinetics
        fib.Ldot = ref_fiber.growth_rate(fib, load, kin.v_grow, kin.stall_force)
        rng = fib.rng if fib.rng is not None else state.rng
        ref_fiber.polymerization_step(fib, dt, rng)
    if state.model("corticalPushing") is not None:
        ref_system.cortical_push_update(state)
    if state.model("cytoplasmicPulling") is not None:
        ref_system.cortical_pull_catastrophe(state)


def _rotation_is_representable(part, omega, dt):
    if float(np.linalg.norm(omega)) * dt < 1e-14:
        return True
    shape = part.mesh.shape
    return shape is not None and shape[0] == "sphere"


def warm_start_vector(state, layout):
    """The current state packed as step unknowns [U omega q1 | q0 | X T]:
    positions X^n for the candidate X^(n+1), the previous step's tensions,
    rigid velocities and densities.  Its residual is O(dt |velocity|), so
    GMRES started there reaches the same relative tolerance (measured
    against the preconditioned rhs, solver.py:459-462) in fewer iterations.
    A device tensor when the state lives on the device (devstate)."""
    from . import devstate
    mirror = devstate.mirror_of(state)
    if mirror is not None:
        return mirror.unknowns_vector(layout)
    x0 = np.zeros(layout.size)
    for i, part in enumerate(state.particles):
        x0[layout.U[i]] = part.U
        x0[layout.omega[i]] = part.omega
        x0[layout.q1[i]] = np.asarray(part.q).ravel()
    if state.periphery is not None:
        x0[layout.q0] = np.asarray(state.periphery.q).ravel()
    for m, fib in enumerate(state.fibers):
        x0[layout.X[m]] = fib.X.ravel()
        x0[layout.T[m]] = fib.T
    return x0


def backward_euler_step(state, dt, params=None, mu=None, backend=None, dt_min=None,
                        implicit_coupling=True, return_info=False, precision="fp64",
                        body_coupling=False, warm_start=False):
    """Advance the state by one implicit step on the device, halving dt on
    nonconvergence (solver.py:528-592).

    The state stays on the device (devstate.DeviceState): the step reads the
    centrelines, tensions, particle meshes and densities from device
    tensors, and writes the solution back into new device tensors (X, T, q,
    U, omega; the particles translate by dt U); the host objects read them
    back only when user code touches them.  Polymerization kinetics and the
    contact models (per-fiber host logic with the reference's RNG draws)
    run only when a fiber is not STALLED or a contact model is configured,
    as in the reference (solver.py:574-588); none of the BASELINE configs
    has either.

    Two options beyond the reference (off by default, same solution to the
    GMRES tolerance): body_coupling=True selects the body-coupled
    preconditioner (see Preconditioner); warm_start=True starts GMRES from
    the current state (warm_start_vector) instead of zero."""
    import torch

    from . import devstate
    from . import fiber as fibers_
    if dt <= 0:
        raise ConfigurationError("time step must be positive")
    if dt_min is None:
        dt_min = dt / 64.0
    attempt = float(dt)
    _native.load(require_device=True)
    mirror = devstate.for_state(state, torch.device("cuda", torch.cuda.current_device()))
    cache = InteractionCache(state, backend=backend, mode=_precision_mode(precision))
    while True:
        op, rhs = assemble_step_operator(state, attempt, mu=mu, backend=backend, cache=cache,
                                         implicit_coupling=implicit_coupling)
        prec = Preconditioner(op, body_coupling=body_coupling)
        x0 = warm_start_vector(state, op.layout) if warm_start else None
        try:
            sol, iters, history = gmres_solve(op, prec, rhs, params, x0=x0)
            break
        except NonconvergenceError as err:
            LOG.warning("step_rejected time=%.9g dt=%.3e residual=%.3e",
                        state.time, attempt, err.residuals[-1])
            if attempt / 2.0 < dt_min:
                raise
            attempt /= 2.0
    lay = op.layout
    # non-spherical particles cannot rotate (their polar parametrisation
    # would break): the reference's check, before any state changes
    for i, part in enumerate(state.particles):
        shape = part.__dict__["_mesh"].shape
        if shape is None or shape[0] != "sphere":
            omega = sol[lay.omega[i]].cpu().numpy()
            if float(np.linalg.norm(omega)) * attempt >= 1e-14:     # _rotation_is_representable
                raise ConfigurationError("rotation of a non-spherical particle is not supported")
    mirror.write_solution(sol, lay, attempt)
    state.time += attempt
    if state.force_models and any(m.kind in ("corticalPushing", "cytoplasmicPulling")
                                  for m in state.force_models) or \
            any(f.growth_state != fibers_.STALLED for f in state.fibers):
        _kinetics_and_contacts(state, attempt)
    LOG.info("step time=%.9g dt=%.3e gmres_iterations=%d residual=%.3e",
             state.time, attempt, iters, history[-1] if history else 0.0)
    if return_info:
        return state, dict(dt=attempt, iterations=iters, history=history, matvecs=op.matvecs)
    return state
