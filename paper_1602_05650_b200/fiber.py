"""Host-side fiber containers mirroring the reference's constructors.

Same names, arguments and validation as slenderflow.fiber
(/root/reference/pkg/src/slenderflow/fiber.py:39-232) so user scripts build
states the same way.  These objects only hold state; every per-step and
per-matvec operation on them runs on the device (operator.py, solver.py).
Geometry is computed lazily on the host for the few host-side consumers
(near-field map construction, attachment wrenches in the API path).
"""

import math
from dataclasses import dataclass

import numpy as np

from . import spectral

GROWING = "growing"
SHRINKING = "shrinking"
STALLED = "stalled"


class InsideFiberError(ValueError):
    pass


@dataclass
class GrowthKinetics:
    """Dynamic-instability parameters (fiber.py:39-48)."""

    v_grow: float = 0.12
    v_shrink: float = 0.288
    f_cat: float = 0.014
    f_res: float = 0.014
    stall_force: float = 4.4
    min_length: float = 0.5


class FreeEnd:
    kind = "free"

    def __repr__(self):
        return "FreeEnd()"


class PrescribedForceTorque:
    kind = "prescribedForceTorque"

    def __init__(self, force, torque=(0.0, 0.0, 0.0)):
        self.force = np.asarray(force, dtype=float)
        self.torque = np.asarray(torque, dtype=float)


class HingedToSurface:
    """Spring attachment of a fiber end to a fixed point (fiber.py:66-75)."""

    kind = "hingedToSurface"

    def __init__(self, attachment, stiffness):
        if stiffness < 0:
            raise ValueError("spring constant must be nonnegative")
        self.attachment = np.asarray(attachment, dtype=float)
        self.stiffness = float(stiffness)


class ClampedToBody:
    """Attachment to a rigid body; tangent=None leaves the end hinged (fiber.py:78-93)."""

    kind = "clampedToBody"

    def __init__(self, body, attach_point, tangent=None):
        self.body = int(body)
        self.attach_point = np.asarray(attach_point, dtype=float)
        if tangent is None:
            self.tangent = None
        else:
            t = np.asarray(tangent, dtype=float)
            nt = np.linalg.norm(t)
            if not np.isclose(nt, 1.0, atol=1e-8):
                raise ValueError("clamped tangent must be a unit vector")
            self.tangent = t / nt


class Fiber:
    """Chebyshev-collocated centreline with tension (fiber.py:96-129).

    Node 0 is the plus end (alpha = +1, s = L), node p the minus end.
    """

    def __init__(self, X, eps, E, delta=None, bc_minus=None, bc_plus=None, tension=None,
                 growth_state=STALLED, Ldot=0.0, rng=None, kinetics=None, tau_cat=math.inf):
        X = np.asarray(X, dtype=float)
        if X.ndim != 2 or X.shape[1] != 3 or X.shape[0] < 5:
            raise ValueError("centerline must be (p+1, 3) with p >= 4")
        if not 0.0 < eps <= 0.1:
            raise ValueError(f"aspect ratio must lie in (0, 0.1], got {eps}")
        if E <= 0:
            raise ValueError("flexural modulus must be positive")
        self._dev = None        # devstate.DeviceState holding this fiber's step unknowns
        self._X = X.copy()
        self._T = np.zeros(X.shape[0]) if tension is None else np.asarray(tension, dtype=float).copy()
        self.eps = float(eps)
        self.E = float(E)
        self.growth_state = growth_state
        self.Ldot = float(Ldot)
        self.bc_minus = bc_minus if bc_minus is not None else FreeEnd()
        self.bc_plus = bc_plus if bc_plus is not None else FreeEnd()
        self.rng = rng
        self.kinetics = kinetics if kinetics is not None else GrowthKinetics()
        self.tau_cat = tau_cat
        self._delta_ratio = None if delta is not None else 0.01
        self._delta = float(delta) if delta is not None else None
        self._geo = None

    # -- geometry (lazy, host) ------------------------------------------------
    # X and T live on the device between implicit steps (devstate.DeviceState):
    # reading them brings the whole state back once, writing them hands the
    # state back to the host (the next step re-uploads it)
    @property
    def X(self):
        if self._dev is not None:
            self._dev.pull()
        return self._X

    @X.setter
    def X(self, value):
        if self._dev is not None:
            self._dev.release()
        self._X = np.asarray(value, dtype=float).copy()
        self._geo = None

    @property
    def T(self):
        if self._dev is not None:
            self._dev.pull()
        return self._T

    @T.setter
    def T(self, value):
        if self._dev is not None:
            self._dev.release()
        self._T = np.asarray(value, dtype=float).copy()

    def refresh_geometry(self):
        s, s_alpha, L, t = spectral.fiber_geometry(self.X, self.p)
        self._geo = dict(s=s, s_alpha=s_alpha, L=L, tangents=t)

    def _g(self, key):
        if self._geo is None:
            self.refresh_geometry()
        return self._geo[key]

    @property
    def s(self):
        return self._g("s")

    @property
    def s_alpha(self):
        return self._g("s_alpha")

    @property
    def L(self):
        return self._g("L")

    @property
    def tangents(self):
        return self._g("tangents")

    @property
    def n_nodes(self):
        return self._X.shape[0]

    @property
    def p(self):
        return self._X.shape[0] - 1

    @property
    def grid(self):
        """ChebyshevGrid of this fiber's order (nodes, weights, D), as in the reference."""
        return spectral.ChebyshevGrid(self.p)

    @property
    def delta(self):
        return self._delta_ratio * self.L if self._delta_ratio is not None else self._delta

    @delta.setter
    def delta(self, value):
        if value <= 0:
            raise ValueError("regularization length must be positive")
        self._delta = float(value)
        self._delta_ratio = None

    @property
    def delta_ratio(self):
        """0.01 for the reference default delta = 0.01 L, None if explicit."""
        return self._delta_ratio

    def end_index(self, plus):
        return 0 if plus else self.p

    def node_weights(self):
        """Quadrature weights converting force density to point strengths (fiber.py:172-174)."""
        return spectral.grid(self.p)[1] * self.s_alpha

    def ds_powers(self):
        """(Ds, Ds2, Ds3) on the host (fiber.py:140-143); API-path helper."""
        D = spectral.grid(self.p)[2]
        Ds = D / self.s_alpha[:, None]
        Ds2 = Ds @ Ds
        return Ds, Ds2, Ds2 @ Ds

    # reference attribute names of the frozen arclength operators (fiber.py:140-143)
    @property
    def Ds(self):
        return self.ds_powers()[0]

    @property
    def Ds2(self):
        return self.ds_powers()[1]

    @property
    def Ds3(self):
        return self.ds_powers()[2]

    @property
    def Ds4(self):
        Ds2 = self.ds_powers()[1]
        return Ds2 @ Ds2

    def copy_state(self):
        return dict(X=self.X.copy(), T=self.T.copy(), L=self.L, Ldot=self.Ldot,
                    growth_state=self.growth_state, tau_cat=self.tau_cat)

    # -- dense per-fiber operators of the reference API (fiber.py:182-222).
    #    The device step never forms these; they serve API users and checks.
    def elastic_operators(self):
        """(FX, FT) with f.ravel() = FX @ X.ravel() + FT @ T."""
        n = self.n_nodes
        Ds, Ds2, _ = self.ds_powers()
        FX = np.zeros((3 * n, 3 * n))
        FT = np.zeros((3 * n, n))
        t = self.tangents
        for c in range(3):
            FX[c::3, c::3] = -self.E * (Ds2 @ Ds2)
            FT[c::3, :] = Ds * t[:, c][None, :]
        return FX, FT

    def mobility_matrix(self, mu):
        """Dense 3n x 3n local mobility, block diagonal over nodes."""
        n = self.n_nodes
        c_log = -math.log(self.eps ** 2 * math.e) / (8.0 * math.pi * mu)
        c_two = 2.0 / (8.0 * math.pi * mu)
        tt = self.tangents[:, :, None] * self.tangents[:, None, :]
        blocks = c_log * (np.eye(3) + tt) + c_two * (np.eye(3) - tt)
        M = np.zeros((3 * n, 3 * n))
        for k in range(n):
            M[3 * k:3 * k + 3, 3 * k:3 * k + 3] = blocks[k]
        return M

    def kdelta_matrix(self, mu):
        """Dense 3n x 3n regularized non-local self-mobility, built by the
        device kernel (bitwise equal to kernels.kdelta_matrix)."""
        from . import kernels
        return kernels.kdelta_matrix(self.X, self.s, self.s_alpha, self.tangents,
                                     spectral.grid(self.p)[1], self.delta,
                                     1.0 / (8.0 * math.pi * mu))


def straight_fiber(p, start, direction, length, eps=0.01, E=10.0, **kwargs):
    """Straight fiber from start along a unit direction; minus end at start (fiber.py:225-232)."""
    d = np.asarray(direction, dtype=float)
    d = d / np.linalg.norm(d)
    s = (spectral.cheb_nodes(p) + 1.0) * (length / 2.0)
    X = np.asarray(start, dtype=float)[None, :] + s[:, None] * d[None, :]
    return Fiber(X, eps=eps, E=E, **kwargs)


def end_force_torque(fib, Xcand, Tcand):
    """Minus-end force and torque on the attached body (fiber.py:361-372), host."""
    Xcand = np.asarray(Xcand, dtype=float)
    Tcand = np.asarray(Tcand, dtype=float)
    k = fib.end_index(plus=False)
    Ds, Ds2, Ds3 = fib.ds_powers()
    Xsss = (Ds3 @ Xcand)[k]
    Xss = (Ds2 @ Xcand)[k]
    t = fib.tangents[k]
    F = -fib.E * Xsss + Tcand[k] * t
    L = fib.E * np.cross(Xss, t)
    return F, L


# -- per-fiber operator API (fiber.py:237-289), evaluated on the device --------

def _dev():
    import torch

    from . import _native
    _native.load(require_device=True)
    return torch.device("cuda")


def _stream():
    import ctypes

    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


def elastic_force_density(fib, Xcand, Tcand):
    """f = -E Ds^4 X + Ds (T X_s) with the geometry frozen (fiber.py:237-241);
    Ds^k built on the device (sf_fiber_dpow), products by the device BLAS."""
    import torch

    from . import _native
    dev = _dev()
    f64 = dict(dtype=torch.float64, device=dev)
    n = fib.n_nodes
    D = torch.tensor(spectral.grid(fib.p)[2], **f64)
    sa = torch.as_tensor(fib.s_alpha, **f64)
    Dpow = torch.empty((1, 4, n, n), **f64)
    _native.call("sf_fiber_dpow", _ptr(D), _ptr(sa), 1, n, _ptr(Dpow), _stream())
    X = torch.as_tensor(np.asarray(Xcand, dtype=float), **f64)
    T = torch.as_tensor(np.asarray(Tcand, dtype=float), **f64)
    t = torch.as_tensor(fib.tangents, **f64)
    f = -fib.E * (Dpow[0, 3] @ X) + Dpow[0, 0] @ (T[:, None] * t)
    return f.cpu().numpy()


def local_mobility_apply(fib, f, mu):
    """(1/8 pi mu)[-ln(eps^2 e)(I + tt) + 2(I - tt)] f (fiber.py:244-250),
    the local half of sf_self_apply_batched."""
    import torch

    from . import _native
    dev = _dev()
    f64 = dict(dtype=torch.float64, device=dev)
    n = fib.n_nodes
    fd = torch.as_tensor(np.asarray(f, dtype=float).reshape(n, 3), **f64).contiguous()
    t = torch.as_tensor(fib.tangents, **f64).contiguous()
    c_log = torch.tensor([-math.log(fib.eps ** 2 * math.e) / (8.0 * math.pi * mu)], **f64)
    u = torch.empty_like(fd)
    _native.call("sf_self_apply_batched", None, _ptr(t), _ptr(c_log), 2.0 / (8.0 * math.pi * mu),
                 _ptr(fd), 1, n, 0, _ptr(u), _stream())
    return u.cpu().numpy()


def nonlocal_Kdelta_apply(fib, f, mu):
    """K_delta f (fiber.py:253-258): K built on the device by
    sf_kdelta_build_batched and applied by sf_self_apply_batched."""
    import torch

    from . import _native
    if fib.delta <= 0:
        raise ValueError("regularization length must be positive")
    dev = _dev()
    f64 = dict(dtype=torch.float64, device=dev)
    n = fib.n_nodes
    X = torch.as_tensor(fib.X, **f64).contiguous()
    s = torch.as_tensor(fib.s, **f64)
    sa = torch.as_tensor(fib.s_alpha, **f64)
    t = torch.as_tensor(fib.tangents, **f64).contiguous()
    w = torch.tensor(spectral.grid(fib.p)[1], **f64)
    delta = torch.tensor([fib.delta], **f64)
    K = torch.empty((1, 3 * n, 3 * n), **f64)
    st = _stream()
    _native.call("sf_kdelta_build_batched", _ptr(X), _ptr(s), _ptr(sa), _ptr(t), _ptr(w), 1, n,
                 _ptr(delta), 1.0 / (8.0 * math.pi * mu), _ptr(K), st)
    fd = torch.as_tensor(np.asarray(f, dtype=float).reshape(n, 3), **f64).contiguous()
    zero = torch.zeros(1, **f64)
    u = torch.empty_like(fd)
    _native.call("sf_self_apply_batched", _ptr(K), _ptr(t), _ptr(zero), 0.0, _ptr(fd), 1, n, 0,
                 _ptr(u), st)
    return u.cpu().numpy()


# -- remaining per-fiber API (fiber.py:26-35, 444-587).  The reference's
#    other host-side per-fiber logic -- the far-field line quadrature
#    fiber_induced_velocity, the dynamic-instability kinetics and the host
#    boundary residuals -- stays in the reference package (_reference.py);
#    the device step assembles the boundary rows analytically (sf_fiber_rows,
#    sf_fiber_self_blocks) ----------------------------------------------------

def shared_grid(p):
    """ChebyshevGrid of order p (fiber.py:26-31)."""
    return spectral.ChebyshevGrid(p)


def resample_to_fine(values, alphas):
    """Chebyshev interpolant of nodal values at new points (fiber.py:444-447)."""
    from numpy.polynomial import chebyshev as C
    return C.chebval(alphas, spectral.cheb_transform(values))


def _plain_map_device(geo, eps, trg, mu, include_doublet):
    """The collocation map (k, 3, 3n) of one fiber at k targets, on the
    device: block j = w_j [S(r) + c D(r)] / (8 pi mu), r = t - x_j, with the
    Stokeslet S = I/r + r r^T/r^3 and, if include_doublet, the doublet
    D = I/r^3 - 3 r r^T/r^5, c = (eps L)^2 / 2 (fiber.py:508-512)."""
    import torch
    X = geo.X[0]
    w = geo.wnode[0]
    r = trg[:, None, :] - X[None, :, :]
    d2 = (r * r).sum(dim=2)
    d = torch.sqrt(d2)
    eye = torch.eye(3, dtype=torch.float64, device=trg.device)
    rr = r[..., :, None] * r[..., None, :]
    K = eye / d[..., None, None] + rr / (d2 * d)[..., None, None]
    if include_doublet:
        c = (eps[0] * geo.L[0]) ** 2 / 2.0
        K = K + c * (eye / (d2 * d)[..., None, None] - 3.0 * rr / (d2 * d2 * d)[..., None, None])
    W = (w[None, :, None, None] * K).permute(0, 2, 1, 3).reshape(trg.shape[0], 3, -1)
    return W / (8.0 * math.pi * mu)


def _one_fiber_geometry(fib):
    import torch

    from .system import FiberGeometry
    ratio = [fib.delta_ratio if fib.delta_ratio is not None else -1.0]
    delta = [0.0 if fib.delta_ratio is not None else fib.delta]
    dev = _dev()
    geo = FiberGeometry(fib.X[None, :, :], ratio, delta, dev)
    return geo, torch.tensor([fib.eps], dtype=torch.float64, device=dev)


def plain_fiber_weights(fib, target, mu, include_doublet=False):
    """Plain collocation map (3, 3n) of one fiber at a target (fiber.py:508-512),
    evaluated on the device."""
    import torch
    geo, eps = _one_fiber_geometry(fib)
    trg = torch.as_tensor(np.asarray(target, dtype=float)[None, :], dtype=torch.float64,
                          device=geo.X.device)
    return _plain_map_device(geo, eps, trg, mu, include_doublet)[0].cpu().numpy()


def near_fiber_weights(fib, target, mu, include_doublet=False):
    """Panel-refined, blended near map (3, 3n) (fiber.py:514-565), built on
    the device: sf_near_fiber_weights gives W_near - W_plain, the plain map
    is added back on the device."""
    import torch

    from . import nearfield
    geo, eps = _one_fiber_geometry(fib)
    trg = torch.as_tensor(np.asarray(target, dtype=float)[None, :], dtype=torch.float64,
                          device=geo.X.device)
    W = nearfield.device_fiber_weights(geo, eps, trg, [0], [0], mu, include_doublet)[0]
    return (W + _plain_map_device(geo, eps, trg, mu, include_doublet)[0]).cpu().numpy()


def near_fiber_eval(fib, f, target, mu, include_doublet=False):
    """Velocity near (but outside) the fiber: near_fiber_weights @ f (fiber.py:576-587)."""
    W = near_fiber_weights(fib, target, mu, include_doublet=include_doublet)
    return W @ np.asarray(f, dtype=float).ravel()
