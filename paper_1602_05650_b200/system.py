"""System state and the complementary-velocity (HI) operator on the B200.

Mirrors the reference's public API (/root/reference/pkg/src/slenderflow/
system.py): SystemState, force models, the SummationBackend plugin,
InteractionCache and complementary_velocities keep their names, arguments,
return types and error behaviour.  The difference is where the work happens:
InteractionCache freezes the geometry ON THE DEVICE (targets, groups,
weights, doublet coefficients, surfaces, particle centres, near-field maps)
and every application is one sf_hi_apply call into libsf_b200.so.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native, nearfield, spectral
from ._native import SF_MODE_FP64
from .fiber import InsideFiberError, end_force_torque
from .kernels import SingularEvaluationError


class ConfigurationError(ValueError):
    pass


class OverlapError(ValueError):
    """A target point lies inside another constituent's volume."""


# -- force models (system.py:40-88) -------------------------------------------

class UniformBodyForce:
    kind = "uniformBodyForce"

    def __init__(self, f0, direction=(0.0, 0.0, 1.0)):
        d = np.asarray(direction, dtype=float)
        nrm = np.linalg.norm(d)
        if nrm == 0.0:
            raise ConfigurationError("load direction must be nonzero")
        self.f0 = float(f0)
        self.direction = d / nrm


class CorticalPushing:
    """Hinged spring attachment of growing plus-ends at the periphery
    (system.py:56-76)."""

    kind = "corticalPushing"

    def __init__(self, stiffness, contact_distance, tau_cat):
        if stiffness < 0 or contact_distance < 0:
            raise ConfigurationError("spring stiffness and contact distance must be nonnegative")
        if tau_cat <= 0:
            raise ConfigurationError("contact catastrophe time must be positive")
        self.stiffness = float(stiffness)
        self.contact_distance = float(contact_distance)
        self.tau_cat = float(tau_cat)


class CytoplasmicPulling:
    kind = "cytoplasmicPulling"

    def __init__(self, motor_force=0.91, motor_density=0.04):
        if motor_force < 0 or motor_density < 0:
            raise ConfigurationError("motor force and density must be nonnegative")
        self.motor_force = float(motor_force)
        self.motor_density = float(motor_density)


# -- summation backend plugin (system.py:93-105) -------------------------------

class DeviceSummation:
    """SummationBackend on the B200: exact pairwise Stokeslet summation.

    Same contract as the reference's DirectSummation: .kind and
    .stokeslet(sources, source_groups, strengths, targets, target_groups, mu)
    -> (Nt,3), raising SingularEvaluationError on a cross-group coincidence.
    """

    kind = "direct"

    def stokeslet(self, sources, source_groups, strengths, targets, target_groups, mu):
        from . import kernels
        out, bad = kernels.stokeslet_sum(targets, target_groups, sources, source_groups,
                                         strengths, 1.0 / (8.0 * np.pi * mu))
        if bad:
            raise SingularEvaluationError(
                "a target coincides with a source outside its own group")
        return out


DirectSummation = DeviceSummation


class TreeSummation:
    """The reference's octree Stokeslet backend (system.py:157-224) on the
    device: same constructor, validation, opening test (theta, analytic
    cell_tolerance gate with C2 = 16) and group-exclusion-by-subtraction;
    the topology is built once per source geometry on the host, moments,
    traversal and leaf sums run in sf_tree_stokeslet.  numpy in -> numpy out,
    CUDA tensors in -> CUDA tensor out."""

    kind = "treeAccelerated"
    _C2 = 16.0

    def __init__(self, theta=0.5, leaf_size=32, cell_tolerance=1e-8):
        if not 0.0 < theta < 1.0:
            raise ConfigurationError("opening parameter must lie in (0, 1)")
        if leaf_size < 1:
            raise ConfigurationError("leaf size must be at least 1")
        if cell_tolerance <= 0:
            raise ConfigurationError("cell tolerance must be positive")
        self.theta = float(theta)
        self.leaf_size = int(leaf_size)
        self.cell_tolerance = float(cell_tolerance)
        self._plans = {}

    def plan(self, sources, source_groups, device=None):
        import torch

        from . import tree
        src = sources.detach().cpu().numpy() if hasattr(sources, "detach") else sources
        grp = source_groups.detach().cpu().numpy() if hasattr(source_groups, "detach") \
            else source_groups
        src = np.asarray(src, dtype=float).reshape(-1, 3)
        key = tree.geometry_key(src, grp, self.leaf_size)
        p = self._plans.pop(key, None)
        if p is None:
            p = tree.TreePlan(src, grp, self.leaf_size, device or torch.device("cuda"))
        self._plans[key] = p
        while len(self._plans) > 2:
            self._plans.pop(next(iter(self._plans)))
        return p

    def stokeslet(self, sources, source_groups, strengths, targets, target_groups, mu):
        import torch
        _native.load(require_device=True)
        dev_io = isinstance(strengths, torch.Tensor) and strengths.is_cuda
        dev = torch.device("cuda")
        p = self.plan(sources, source_groups, dev)
        f64 = dict(dtype=torch.float64, device=dev)
        f = torch.as_tensor(strengths, **f64).reshape(-1, 3).contiguous()
        t = torch.as_tensor(targets, **f64).reshape(-1, 3).contiguous()
        tg = torch.as_tensor(target_groups, dtype=torch.int64, device=dev).contiguous()
        out = p.stokeslet(f, t, tg, mu, self.theta, self.cell_tolerance)
        return out if dev_io else out.cpu().numpy()


# -- state (system.py:237-278) -------------------------------------------------

class SystemState:
    """The constituents, fluid viscosity, force models and clock of a
    simulation: the reference's SystemState constructor and invariants
    (system.py:237-278).  Between implicit steps the constituents' unknowns
    live on the device (devstate.DeviceState, attached as `_dev`)."""

    def __init__(self, fibers, particles=(), periphery=None, mu=1.0, time=0.0,
                 force_models=(), seed=None):
        if mu <= 0:
            raise ConfigurationError("viscosity must be positive")
        self.fibers, self.particles = list(fibers), list(particles)
        self.periphery, self.force_models = periphery, list(force_models)
        self.mu, self.time, self.seed = float(mu), float(time), seed
        self.rng = np.random.default_rng(seed)
        self.validate()

    def validate(self):
        """Raise ConfigurationError on the first violated invariant, checked
        in the reference's order: constituents inside the periphery (one
        batched containment test per family), then each fiber's boundary
        conditions."""
        per = self.periphery
        if per is not None:
            for what, pts in (("fiber", [f.X for f in self.fibers]),
                              ("particle", [p.mesh.nodes for p in self.particles])):
                if not pts:
                    continue
                owner = np.repeat(np.arange(len(pts)), [len(x) for x in pts])
                outside = ~per.contains(np.concatenate(pts))
                if outside.any():
                    leave = "leaves the confining periphery"
                    raise ConfigurationError(f"{what} {owner[np.argmax(outside)]} {leave}")
        nparts = len(self.particles)
        for i, fib in enumerate(self.fibers):
            if fib.bc_plus.kind == "clampedToBody":
                raise ConfigurationError("plus-end clamping is not supported")
            for bc in (fib.bc_minus, fib.bc_plus):
                if bc.kind == "clampedToBody" and not 0 <= bc.body < nparts:
                    raise ConfigurationError(f"fiber {i} is clamped to a body outside the system")
                if bc.kind == "hingedToSurface" and per is None:
                    raise ConfigurationError(
                        f"fiber {i} is hinged to a surface but no periphery is present")

    def model(self, kind):
        """First configured force model of `kind`, or None."""
        return next((m for m in self.force_models if m.kind == kind), None)


def external_force_density(state, fib):
    """Per-node external force density from the force models (system.py:297-305)."""
    f = np.zeros((fib.n_nodes, 3))
    for m in state.force_models:
        if m.kind == "uniformBodyForce":
            f += m.f0 * m.direction[None, :]
        elif m.kind == "cytoplasmicPulling":
            f += m.motor_force * m.motor_density * fib.tangents
    return f


def attachment_wrench(state, particle_index, candidates=None):
    """Net force and torque on a particle from its clamped fibers (system.py:308-329)."""
    part = state.particles[particle_index]
    F = np.zeros(3)
    L = np.zeros(3)
    for k, fib in enumerate(state.fibers):
        bc = fib.bc_minus
        if bc.kind != "clampedToBody" or bc.body != particle_index:
            continue
        cand = None if candidates is None else candidates[k]
        X, T = (fib.X, fib.T) if cand is None else cand
        Fe, Le = end_force_torque(fib, X, T)
        arm = fib.X[fib.end_index(plus=False)] - part.center
        F += Fe
        L += Le + np.cross(arm, Fe)
    return F, L


@dataclass
class ComplementaryVelocities:
    periphery: object
    particles: list
    fibers: list


def _inside_star_surface(mesh, points):
    pts = np.atleast_2d(points) - mesh.center
    rho = np.linalg.norm(pts, axis=1)
    safe = np.where(rho > 0, rho, 1.0)
    th = np.arccos(np.clip(np.where(rho > 0, pts[:, 2] / safe, 1.0), -1.0, 1.0))
    return rho < np.asarray(mesh.shape[2](th), dtype=float)


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def stack_fibers(fibers):
    """(nf, n, 3) centrelines of fibers that share one node count."""
    if not fibers:
        return np.zeros((0, 5, 3))
    n = fibers[0].n_nodes
    if any(f.n_nodes != n for f in fibers):
        raise ConfigurationError("stack_fibers needs every fiber to have the same order p")
    return np.stack([f.X for f in fibers])


def order_classes(fibers):
    """[(n, idx)]: the fibers grouped by node count (Chebyshev order), each
    class a uniform batch for the per-fiber kernels; idx ascending."""
    ns = np.array([f.n_nodes for f in fibers], dtype=np.int64)
    out = []
    for n in dict.fromkeys(ns.tolist()):
        out.append((int(n), np.nonzero(ns == n)[0]))
    return out


class FiberGeometry:
    """Batched per-fiber geometry on the device (sf_fiber_geometry_batched)."""

    def __init__(self, X, delta_ratio, delta, device):
        import torch
        dev = dict(dtype=torch.float64, device=device)
        X = torch.as_tensor(X, **dev).contiguous()
        nf, n, _ = X.shape
        self.nf, self.n = nf, n
        _, wcc, D, S = spectral.grid(n - 1)
        self.X = X
        self.wcc = torch.tensor(wcc, **dev)
        self.D = torch.tensor(D, **dev)
        self.S = torch.tensor(S, **dev)
        self.s = torch.empty((nf, n), **dev)
        self.s_alpha = torch.empty((nf, n), **dev)
        self.tang = torch.empty((nf, n, 3), **dev)
        self.wnode = torch.empty((nf, n), **dev)
        self.L = torch.empty(nf, **dev)
        self.delta = torch.as_tensor(np.asarray(delta, dtype=float), **dev).clone()
        degenerate = torch.zeros(1, dtype=torch.int32, device=device)
        if nf:
            _native.call("sf_fiber_geometry_batched", _ptr(X), nf, n, _ptr(self.D), _ptr(self.S),
                         _ptr(self.wcc), -1.0, _ptr(self.s), _ptr(self.s_alpha), _ptr(self.tang),
                         _ptr(self.wnode), _ptr(self.L), None, _ptr(degenerate), _stream())
            if int(degenerate.item()):
                raise ValueError("centerline parametrization is degenerate")
            # delta = ratio * L where the fiber uses the default ratio (fiber.py:127,144)
            ratio = torch.as_tensor(np.asarray(delta_ratio, dtype=float), **dev)
            self.delta = torch.where(ratio > 0, ratio * self.L, self.delta)


class _DeviceMesh:
    """A moving rigid particle's mesh while its nodes live on the device:
    the static attributes (normals, weights, parametrisation, shape) of the
    host mesh, the current nodes and centre as device tensors, host copies
    of those read back on demand."""

    def __init__(self, base, nodes_dev, center_dev):
        self.base = base
        self.nodes_dev = nodes_dev
        self.center_dev = center_dev
        for a in ("normals", "weights", "thetas", "phis", "patch_grid", "shape", "area", "h"):
            setattr(self, a, getattr(base, a))
        self._nodes = self._center = None

    @property
    def n_nodes(self):
        return self.base.n_nodes

    def has_parametrization(self):
        return self.base.has_parametrization()

    def surface_point(self, theta, phi):
        R = self.shape[2](theta)
        st = np.sin(theta)
        return self.center + R * np.array([st * np.cos(phi), st * np.sin(phi), np.cos(theta)])

    def radial_bound(self, theta):
        return float(self.shape[2](theta))

    def refined(self, factor):
        from .body import make_surface
        nt, nph = self.patch_grid
        return make_surface(self.shape, (nt * factor, nph * factor), center=self.center)

    @property
    def nodes(self):
        if self._nodes is None:
            self._nodes = self.nodes_dev.cpu().numpy()
        return self._nodes

    @property
    def center(self):
        if self._center is None:
            self._center = self.center_dev.cpu().numpy()
        return self._center


class InteractionCache:
    """Frozen-geometry layout of complementary_velocities, resident on the B200
    (system.py:492-620).  Rebuild whenever any constituent moves."""

    def __init__(self, state, include_doublet=True, device=None, mode=SF_MODE_FP64,
                 near="device", fiber_geometry=None, target_range=None, fiber_pairs=True,
                 backend=None):
        """target_range (lo, hi): evaluate only the targets [lo, hi) of the
        global [particles | periphery | fibers] list (a rank's share in a
        multi-GPU step).  fiber_pairs=False leaves the fiber-source pair sum
        out of the layout (evaluated elsewhere, e.g. symmetrically across
        ranks); the near corrections of fiber sources stay in."""
        import os
        import time

        import torch
        _dbg = os.environ.get("SF_DEBUG_TIMING")
        _t = [time.perf_counter()]

        def _lap(label):
            if _dbg:
                torch.cuda.synchronize()
                now = time.perf_counter()
                print(f"  cache {label:28s} {1e3 * (now - _t[0]):9.2f} ms", flush=True)
                _t[0] = now
        from . import devstate
        # the step's state on the device (devstate.DeviceState): targets,
        # fiber geometry and surfaces come from its tensors, not the host
        mirror = devstate.mirror_of(state) if fiber_geometry is None else None
        self.mirror = mirror
        if mirror is not None:
            self.device = mirror.device
        else:
            self.device = torch.device(device) if device is not None else torch.device("cuda")
        dev = dict(device=self.device)
        f64 = dict(dtype=torch.float64, **dev)
        self.include_doublet = include_doublet
        self.mu = state.mu
        nf = len(state.fibers)
        np_ = len(state.particles)
        self.nf, self.np = nf, np_

        # surfaces: particles then periphery (system.py:544-557); moving
        # particle meshes are device-backed views while a mirror is live
        self.surfaces = []
        surf_dev = []
        for i, part in enumerate(state.particles):
            if mirror is not None:
                mesh = _DeviceMesh(part.__dict__["_mesh"], mirror.pnodes[i], mirror.pmesh_center[i])
                surf_dev.append((mesh.nodes_dev, mirror.pnrm[i], mirror.pw[i]))
            else:
                mesh = part.mesh
                surf_dev.append(None)
            self.surfaces.append((mesh, nf + i, False))
        if state.periphery is not None:
            self.surfaces.append((state.periphery.mesh, nf + np_, True))
            surf_dev.append((mirror.per_nodes, mirror.per_nrm, mirror.per_w)
                            if mirror is not None else None)
        self.surface_arrays = [
            sd if sd is not None else (torch.as_tensor(m.nodes, **f64),
                                       torch.as_tensor(m.normals, **f64),
                                       torch.as_tensor(m.weights, **f64))
            for sd, (m, _, _) in zip(surf_dev, self.surfaces)]

        groups = []
        self.particle_slices = []
        off = 0
        for i, part in enumerate(state.particles):
            n = self.surfaces[i][0].n_nodes
            groups.append(np.full(n, nf + i, dtype=np.int64))
            self.particle_slices.append(slice(off, off + n))
            off += n
        self.periphery_slice = None
        if state.periphery is not None:
            n = state.periphery.mesh.n_nodes
            groups.append(np.full(n, nf + np_, dtype=np.int64))
            self.periphery_slice = slice(off, off + n)
            off += n
        # fibers in order; node counts may differ (mixed Chebyshev orders)
        ns = np.array([f.n_nodes for f in state.fibers], dtype=np.int64)
        self.node_counts = ns
        self.pt_off = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64) if nf else ns
        self.uniform = len(set(ns.tolist())) <= 1
        self.n_nodes = int(ns[0]) if (nf and self.uniform) else (5 if not nf else 0)
        npts = int(ns.sum())
        self.fiber_slice = slice(off, off + npts)
        self.fiber_slices = [slice(off + int(self.pt_off[m]), off + int(self.pt_off[m] + ns[m]))
                             for m in range(nf)]
        groups.append(np.repeat(np.arange(nf, dtype=np.int64), ns))
        self.target_groups = np.concatenate(groups) if groups else np.zeros(0, np.int64)
        # target positions [particles | periphery | fibers], on the device
        tblocks = [a[0] for a in self.surface_arrays]
        if mirror is not None:
            fx = torch.empty((npts, 3), **f64)
            for n, idx, X in mirror.fiber_X():
                pidx = torch.as_tensor((self.pt_off[idx][:, None] + np.arange(n)).reshape(-1), **dev)
                fx[pidx] = X.reshape(-1, 3)
            tblocks.append(fx)
        else:
            tblocks.append(torch.as_tensor(np.concatenate([f.X for f in state.fibers]) if nf
                                           else np.zeros((0, 3)), **f64))
        trg = torch.cat(tblocks) if len(tblocks) > 1 else tblocks[0]
        self._targets_host = None
        self.target_offset = 0
        if target_range is not None:
            lo, hi = target_range
            trg = trg[lo:hi]
            self.target_groups = self.target_groups[lo:hi]
            self.target_offset = lo

            def clip(sl):
                a, b = max(sl.start, lo), min(sl.stop, hi)
                return slice(a - lo, b - lo) if a < b else slice(0, 0)
            self.particle_slices = [clip(x) for x in self.particle_slices]
            if self.periphery_slice is not None:
                self.periphery_slice = clip(self.periphery_slice)
            self.fiber_slice = clip(self.fiber_slice)
            self.fiber_slices = [clip(x) for x in self.fiber_slices]
        self.trg = trg.contiguous()
        self.n_targets = self.trg.shape[0]
        kind = getattr(backend, "kind", "direct") if backend is not None else "direct"
        if kind not in ("direct", "treeAccelerated"):
            raise ConfigurationError(f"backend {kind!r} is not available on the device")
        # tree backend: the fiber Stokeslet goes through the octree, the
        # doublet stays a direct sum (system.py:659-671)
        self.backend = backend if kind == "treeAccelerated" else None
        self.fiber_pairs = bool(fiber_pairs) and self.backend is None

        _lap("targets")
        # fibers: geometry, weights, doublet coefficients (device), one
        # batched FiberGeometry per order class, flat point arrays in fiber order
        self.eps = torch.as_tensor([f.eps for f in state.fibers], **f64)
        if fiber_geometry is not None:
            self.classes = [(self.n_nodes, np.arange(nf), fiber_geometry)]
        elif nf == 0:
            self.classes = [(5, np.arange(0), FiberGeometry(np.zeros((0, 5, 3)), [], [],
                                                            self.device))]
        else:
            self.classes = []
            Xdev = {n: X for n, _, X in mirror.fiber_X()} if mirror is not None else None
            for n, idx in order_classes(state.fibers):
                fibs = [state.fibers[m] for m in idx]
                ratios = [f.delta_ratio if f.delta_ratio is not None else -1.0 for f in fibs]
                deltas = [0.0 if f.delta_ratio is not None else f.delta for f in fibs]
                X = Xdev[n] if Xdev is not None else stack_fibers(fibs)
                self.classes.append((n, idx, FiberGeometry(X, ratios, deltas, self.device)))
        self.geo = self.classes[0][2] if (self.uniform and self.classes) else None
        if self.geo is not None:
            self.fsrc = self.geo.X.reshape(-1, 3)
            self.fw = self.geo.wnode.reshape(-1)
            self.fL = self.geo.L
        else:
            self.fsrc = torch.empty((npts, 3), **f64)
            self.fw = torch.empty(npts, **f64)
            self.fL = torch.empty(nf, **f64)
            for n, idx, g in self.classes:
                pidx = torch.as_tensor((self.pt_off[idx][:, None] + np.arange(n)).reshape(-1),
                                       **dev)
                self.fsrc[pidx] = g.X.reshape(-1, 3)
                self.fw[pidx] = g.wnode.reshape(-1)
                self.fL[torch.as_tensor(idx, **dev)] = g.L
        self.fgrp = torch.as_tensor(np.repeat(np.arange(nf, dtype=np.int64), ns), **dev)
        self.fdcoef = (((self.eps * self.fL) ** 2 / 2.0).repeat_interleave(
            torch.as_tensor(ns, **dev)) if include_doublet and nf else None)   # system.py:542

        self.surface_offsets = []
        o = 0
        for m, _, _ in self.surfaces:
            self.surface_offsets.append(o)
            o += m.n_nodes
        self.nss = o
        if self.surfaces:
            self.ssrc = torch.cat([a[0] for a in self.surface_arrays]).contiguous()
            self.snrm = torch.cat([a[1] for a in self.surface_arrays]).contiguous()
            self.sw = torch.cat([a[2] for a in self.surface_arrays]).contiguous()
            self.sgrp = torch.as_tensor(np.concatenate(
                [np.full(m.n_nodes, g, dtype=np.int64) for m, g, _ in self.surfaces]), **dev)
        else:
            self.ssrc = self.snrm = self.sw = self.sgrp = None
        if mirror is not None:
            self.pcenter = mirror.pcenter if np_ else None
        else:
            self.pcenter = (torch.as_tensor(np.stack([p.center for p in state.particles]), **f64)
                            if np_ else None)
        self.tgrp = torch.as_tensor(self.target_groups, **dev)
        self.pgrp = torch.as_tensor(np.arange(nf, nf + np_, dtype=np.int64), **dev) if np_ else None

        _lap("geometry + surfaces")
        self._check_surface_overlaps()
        _lap("overlap checks")
        # near maps: fibers on the device (default) or the host restatement
        self._near_fiber_list = []
        self._near_dev = None
        if near not in (None, False, "device"):
            raise ConfigurationError("near-field maps are built on the device (near='device')")
        if near and nf:
            try:
                if self.uniform:
                    t, l, W = nearfield.device_fiber_pairs(self.geo, self.eps, self.trg, self.tgrp,
                                                           state.mu, include_doublet)
                    self._near_dev = (t, l, W)
                    self._near_fiber_list = None      # built on first access (near_fiber)
                else:
                    self._near_fiber_list = self._class_near_pairs(state.mu, include_doublet)
            except InsideFiberError as err:
                raise OverlapError(f"target node overlaps a fiber: {err}") from err
        _lap("near fiber maps")
        self.near_surface = []
        if near and self.surfaces:
            self.near_surface = nearfield.device_surface_pairs(
                self.surfaces, self.trg, self.tgrp, state.mu, self.device,
                surface_arrays=self.surface_arrays)
        _lap("near surface maps")
        self._build_near_map()
        _lap("near CSR")
        self.mode = int(mode)
        self._layout()
        self.bad = torch.zeros(3, dtype=torch.int64, **dev)

    # -- the reference's host-side attributes (system.py:536-557), read back
    #    from the device layout on demand --------------------------------------
    @property
    def near_fiber(self):
        """[(target, fiber, W (3, 3n))] in the reference's order
        (system.py:564-599); device-built maps are listed on first access
        (the step itself uses the device arrays directly)."""
        if self._near_fiber_list is None:
            t, l, W = self._near_dev
            self._near_fiber_list = list(zip(t.tolist(), l.tolist(), W))
        return self._near_fiber_list

    @property
    def fiber_sources(self):
        return self.fsrc.cpu().numpy()

    @property
    def fiber_groups(self):
        return self.fgrp.cpu().numpy()

    @property
    def fiber_weights(self):
        return np.split(self.fw.cpu().numpy(), np.cumsum(self.node_counts)[:-1])

    @property
    def doublet_coeffs(self):
        return list(((self.eps * self.fL) ** 2 / 2.0).cpu().numpy())

    @property
    def surface_sources(self):
        return self.ssrc.cpu().numpy() if self.ssrc is not None else np.zeros((0, 3))

    @property
    def surface_normals(self):
        return self.snrm.cpu().numpy() if self.snrm is not None else np.zeros((0, 3))

    @property
    def surface_groups(self):
        return self.sgrp.cpu().numpy() if self.sgrp is not None else np.zeros(0, dtype=np.int64)

    # -- construction helpers ------------------------------------------------
    def _class_near_pairs(self, mu, include_doublet):
        """Device near maps of a mixed-order system, one order class at a
        time (target groups remapped so only a fiber's own nodes are
        excluded), merged in the reference's order (fiber, then target)."""
        import torch
        entries = []
        nf = self.nf
        for n, idx, g in self.classes:
            loc = np.full(nf + self.np + 2, -1, dtype=np.int64)
            loc[idx] = np.arange(idx.size)
            tg = loc[np.clip(self.target_groups, -1, nf + self.np + 1)]
            tg[self.target_groups < 0] = -1
            t, l, W = nearfield.device_fiber_pairs(
                g, self.eps[torch.as_tensor(idx, device=self.device)], self.trg,
                torch.as_tensor(tg, device=self.device), mu, include_doublet)
            entries.extend(zip(t.tolist(), idx[l].tolist(), W))
        entries.sort(key=lambda e: (e[1], e[0]))
        return entries


    @property
    def targets(self):
        """Target positions (n_targets, 3) on the host (read back on demand;
        the device path uses trg)."""
        if self._targets_host is None:
            self._targets_host = self.trg.cpu().numpy()
        return self._targets_host

    def _check_surface_overlaps(self):
        """Targets of other constituents inside a rigid particle or outside
        the periphery raise OverlapError (system.py:581-583, 591-598).  Sphere
        meshes are tested on the device (rho < R, one flag read for all
        surfaces); other star-shaped profiles on the host."""
        import torch
        flags = []
        for si, (mesh, group, is_periphery) in enumerate(self.surfaces):
            if mesh.shape is None:
                continue
            if mesh.shape[0] == "sphere":
                center = getattr(mesh, "center_dev", None)
                if center is None:
                    center = torch.as_tensor(mesh.center, dtype=torch.float64, device=self.device)
                rho = torch.linalg.vector_norm(self.trg - center, dim=1)
                inside = rho < float(mesh.shape[1])
                bad = (self.tgrp != group) & (~inside if is_periphery else inside)
                flags.append(bad.any())
                continue
            others = self.target_groups != group
            inside = _inside_star_surface(mesh, self.targets)
            flags.append(torch.tensor(bool(np.any(others & ~inside) if is_periphery
                                           else np.any(others & inside)), device=self.device))
        if not flags:
            return
        hit = torch.stack(flags).cpu().numpy()
        for f, (mesh, group, is_periphery) in zip(hit, [x for x in self.surfaces
                                                        if x[0].shape is not None]):
            if f:
                raise OverlapError("a target lies outside the confining periphery" if is_periphery
                                   else "a target lies inside a rigid particle")

    def _build_near_map(self):
        """CSR by target of every correction map, fiber entries before surface
        entries for a target (the reference applies the fiber list first,
        system.py:702-707).  x = [fiber forces | surface densities], flattened.
        Map matrices stay where they were built (fiber maps in one device
        block, then the surface maps); entries address them by offset."""
        import torch
        self.near_nrows = 0
        self.near_tensors = {}
        nfs3 = 3 * int(self.node_counts.sum())
        dev = dict(device=self.device)
        f64 = dict(dtype=torch.float64, **dev)
        blocks, wo_parts = [], []
        if self._near_dev is not None:
            t_d, l_d, W_d = self._near_dev
            tf = np.asarray(t_d.cpu().numpy() if torch.is_tensor(t_d) else t_d, dtype=np.int64)
            lf = np.asarray(l_d.cpu().numpy() if torch.is_tensor(l_d) else l_d, dtype=np.int64)
            if tf.size:
                per = int(W_d[0].numel())
                blocks.append(W_d.reshape(-1))
                wo_parts.append(np.arange(tf.size, dtype=np.int64) * per)
        else:
            nearf = self._near_fiber_list
            tf = np.array([e[0] for e in nearf], dtype=np.int64)
            lf = np.array([e[1] for e in nearf], dtype=np.int64)
            pieces = [torch.as_tensor(e[2], **f64).reshape(-1) for e in nearf]
            if pieces:
                sizes = np.array([x.numel() for x in pieces], dtype=np.int64)
                wo_parts.append(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64))
                blocks.append(torch.cat(pieces))
        base = int(sum(b.numel() for b in blocks))
        ns = self.near_surface
        ts = np.array([e[0] for e in ns], dtype=np.int64)
        ls = np.array([e[1] for e in ns], dtype=np.int64)
        if ns:
            pieces = [torch.as_tensor(e[2], **f64).reshape(-1) for e in ns]
            sizes = np.array([x.numel() for x in pieces], dtype=np.int64)
            wo_parts.append(base + np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64))
            blocks.append(torch.cat(pieces))
        t = np.concatenate([tf, ts])
        if t.size == 0:
            return
        s_off = np.asarray(self.surface_offsets, dtype=np.int64) if ns else np.zeros(0, np.int64)
        s_n = (np.array([m.n_nodes for m, _, _ in self.surfaces], dtype=np.int64) if ns
               else np.zeros(0, np.int64))
        xo = np.concatenate([3 * self.pt_off[lf], nfs3 + 3 * s_off[ls] if ns else ls])
        xl = np.concatenate([3 * self.node_counts[lf], 3 * s_n[ls] if ns else ls])
        wo = np.concatenate(wo_parts)
        order = np.argsort(t, kind="stable")
        t = t[order]
        rows, starts = np.unique(t, return_index=True)
        self.near_tensors = dict(
            row_ptr=torch.as_tensor(np.append(starts, t.size).astype(np.int64), **dev),
            rows=torch.as_tensor(rows, **dev),
            w_off=torch.as_tensor(wo[order], **dev),
            x_off=torch.as_tensor(xo[order].astype(np.int64), **dev),
            x_len=torch.as_tensor(xl[order].astype(np.int64), **dev),
            W=(torch.cat(blocks) if len(blocks) > 1 else blocks[0]).contiguous())
        self.near_nrows = rows.size

    def _layout(self):
        nt = self.near_tensors
        nfs = self.fsrc.shape[0] if self.fiber_pairs else 0
        whole = self.target_offset == 0 and self.fiber_slice.stop == self.n_targets and \
            self.fiber_slice.stop - self.fiber_slice.start == self.fsrc.shape[0]
        self.layout = _native.HiLayout(
            trg=_ptr(self.trg), tgrp=_ptr(self.tgrp), nt=self.n_targets,
            fsrc=_ptr(self.fsrc), fgrp=_ptr(self.fgrp), fw=_ptr(self.fw),
            fdcoef=_ptr(self.fdcoef), nfs=nfs,
            ssrc=_ptr(self.ssrc), snrm=_ptr(self.snrm), sw=_ptr(self.sw), sgrp=_ptr(self.sgrp),
            nss=self.nss, pcenter=_ptr(self.pcenter), pgrp=_ptr(self.pgrp), np=self.np,
            near_row_ptr=_ptr(nt.get("row_ptr")), near_rows=_ptr(nt.get("rows")),
            near_w_off=_ptr(nt.get("w_off")), near_x_off=_ptr(nt.get("x_off")),
            near_x_len=_ptr(nt.get("x_len")), near_nrows=self.near_nrows,
            near_W=_ptr(nt.get("W")), mu=self.mu, mode=self.mode,
            fiber_target_off=self.fiber_slice.start if (self.nf and whole) else -1,
            fiber_group_size=self.n_nodes if self.uniform else 0)

    # -- application ------------------------------------------------------------
    @property
    def pairs_per_apply(self):
        """Non-excluded (target, source) pairs of one application."""
        nfs = self.fsrc.shape[0] if self.fiber_pairs else 0
        ln = lambda sl: sl.stop - sl.start                                 # noqa: E731
        own = (sum(ln(s) * int(n) for s, n in zip(self.fiber_slices, self.node_counts))
               if self.fiber_pairs else 0)
        tsl = list(self.particle_slices) + ([self.periphery_slice]
                                             if self.periphery_slice is not None else [])
        surf = sum(ln(s) * m.n_nodes for s, (m, _, _) in zip(tsl, self.surfaces))
        return self.n_targets * nfs - own + self.n_targets * self.nss - surf

    def apply(self, f, q=None, wrench=None, out=None, check=True):
        """u (n_targets,3) on the device; f (nfs,3), q (nss,3), wrench (np,6)."""
        import torch
        f64 = dict(dtype=torch.float64, device=self.device)
        f = torch.as_tensor(f, **f64).reshape(-1, 3).contiguous()
        if q is not None:
            q = torch.as_tensor(q, **f64).reshape(-1, 3).contiguous()
        if wrench is not None:
            wrench = torch.as_tensor(wrench, **f64).reshape(-1, 6).contiguous()
        if out is None:
            out = torch.empty((self.n_targets, 3), **f64)
        x = None
        if self.near_nrows:
            x = f.reshape(-1) if q is None else torch.cat([f.reshape(-1), q.reshape(-1)])
        _native.call("sf_hi_apply", ctypes.byref(self.layout), _ptr(f), _ptr(q), _ptr(wrench),
                     _ptr(x), _ptr(out), _ptr(self.bad), _stream())
        if check:
            self.check_bad()
        if self.backend is not None and self.nf and self.n_targets:
            self._tree_fiber_terms(f, out)
        return out

    def _tree_fiber_terms(self, f, out):
        """Fiber Stokeslet through the tree backend + direct doublet
        (complementary_velocities, system.py:655-671)."""
        import torch
        s = self.fw[:, None] * f
        if getattr(self, "_tree_plan", None) is None:      # topology once per geometry
            self._tree_plan = self.backend.plan(self.fsrc, self.fgrp, self.device)
        b = self.backend
        out += self._tree_plan.stokeslet(s, self.trg, self.tgrp, self.mu, b.theta, b.cell_tolerance)
        if self.fdcoef is not None:
            dbl = (self.fdcoef[:, None] * s).contiguous()
            tmp = torch.empty_like(out)
            bad = torch.zeros(1, dtype=torch.int64, device=self.device)
            _native.call("sf_doublet_sum", _ptr(self.trg), _ptr(self.tgrp), self.n_targets,
                         _ptr(self.fsrc), _ptr(self.fgrp), self.fsrc.shape[0], _ptr(dbl),
                         1.0 / (8.0 * math.pi * self.mu), _ptr(tmp), _ptr(bad), _stream())
            if int(bad.item()):
                raise SingularEvaluationError("a target coincides with another fiber's node")
            out += tmp

    def check_bad(self):
        b = self.bad.tolist()
        if b[0]:
            raise SingularEvaluationError("a target coincides with another fiber's node")
        if b[1]:
            raise SingularEvaluationError("a target coincides with another surface's node")
        if b[2]:
            raise SingularEvaluationError("target at a particle center")

    def split(self, u):
        """Break a stacked velocity array into the evaluation families (system.py:615-620)."""
        per = u[self.periphery_slice] if self.periphery_slice is not None else None
        return ComplementaryVelocities(periphery=per,
                                       particles=[u[s] for s in self.particle_slices],
                                       fibers=[u[s] for s in self.fiber_slices])


def complementary_velocities(state, periphery_density=None, particle_densities=None,
                             fiber_forces=None, particle_wrenches=None, backend=None, cache=None,
                             include_doublet=True):
    """Flow induced at every constituent's nodes by all the others (system.py:623-709).

    Same signature and results as the reference; the evaluation runs on the
    B200 through the (device-resident) InteractionCache.  Host (numpy)
    inputs give numpy outputs.
    """
    if cache is None:
        cache = InteractionCache(state, include_doublet=include_doublet, backend=backend)
    if fiber_forces is None:
        from .fiber import elastic_force_density
        fiber_forces = [elastic_force_density(f, f.X, f.T) + external_force_density(state, f)
                        for f in state.fibers]
    if particle_densities is None:
        particle_densities = [p.q for p in state.particles]
    if periphery_density is None and state.periphery is not None:
        periphery_density = state.periphery.q
    if particle_wrenches is None:
        particle_wrenches = []
        for i, part in enumerate(state.particles):
            Fa, La = attachment_wrench(state, i)
            particle_wrenches.append((part.F_ext + Fa, part.L_ext + La))
    f = (np.concatenate([np.asarray(x, dtype=float).reshape(-1, 3) for x in fiber_forces])
         if state.fibers else np.zeros((0, 3)))
    q = None
    if cache.surfaces:
        q = np.concatenate([np.asarray(periphery_density if isp else particle_densities[j],
                                       dtype=float).reshape(-1, 3)
                            for j, (_, _, isp) in enumerate(cache.surfaces)])
    w = None
    if state.particles:
        w = np.concatenate([np.concatenate([np.asarray(F, dtype=float), np.asarray(L, dtype=float)])
                            for F, L in particle_wrenches])
    u = cache.apply(f, q, w).cpu().numpy()
    return cache.split(u)
