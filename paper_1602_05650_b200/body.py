"""Host-side surface containers and mesh setup (body.py of the reference).

Surfaces of revolution quadrangulated on a uniform (theta, phi) patch grid
with a 4x4 tensor Gauss-Legendre rule per patch -- the reference's
discretisation (/root/reference/pkg/src/slenderflow/body.py:127-184), so the
same `make_surface(shape, resolution)` call yields the same nodes, normals
and weights.  Mesh generation is one-time host setup; the layer potentials
evaluated on these meshes run on the device (operator.py / solver.py).
"""

import math

import numpy as np

_GL_X, _GL_W = np.polynomial.legendre.leggauss(4)
GL01_NODES = 0.5 * (_GL_X + 1.0)
GL01_WEIGHTS = 0.5 * _GL_W
NEAR_SHELL_FACTOR = 1.5


class GeometryError(ValueError):
    pass


def sphere_shape(radius):
    if radius <= 0:
        raise GeometryError("sphere radius must be positive")
    r = float(radius)
    return ("sphere", r, lambda th: np.full_like(np.asarray(th, dtype=float), r),
            lambda th: np.zeros_like(np.asarray(th, dtype=float)))


def _profile(name, a, R, Rp):
    return (name, a, R, Rp)


def s1_shape(a):
    """Asymmetric cell profile of the reference (body.py:37-41)."""
    c3 = lambda th: np.cos(th) ** 3                                     # noqa: E731
    s3 = lambda th: np.sin(th) ** 3                                     # noqa: E731
    return _profile("s1", a, lambda th: a * (1.0 - 0.35 * c3(th) - 0.15 * s3(th)),
                    lambda th: a * (1.05 * np.cos(th) ** 2 * np.sin(th)
                                    - 0.45 * np.sin(th) ** 2 * np.cos(th)))


def s2_shape(a):
    """Tilted-ellipsoid-like profile (body.py:44-47)."""
    return _profile("s2", a, lambda th: a * (1.0 + 0.2 * np.cos(2 * th) - 0.2 * np.sin(2 * th)),
                    lambda th: a * (-0.4 * np.sin(2 * th) - 0.4 * np.cos(2 * th)))


def s3_shape(a):
    """Flattened (oblate) profile (body.py:50-53)."""
    return _profile("s3", a, lambda th: a * (1.0 - 0.6 * np.sin(th) ** 4),
                    lambda th: a * (-2.4 * np.sin(th) ** 3 * np.cos(th)))


def profile_shape(R, Rp=None, name="profile", param=0.0):
    """User profile R(theta); Rp by central differences when omitted (body.py:56-60)."""
    if Rp is None:
        def Rp(th, _R=R, h=1e-5):
            th = np.asarray(th)
            return (_R(th + h) - _R(th - h)) / (2 * h)
    return (name, param, R, Rp)


_NAMED = {"s1": s1_shape, "s2": s2_shape, "s3": s3_shape}


def named_shape(kind, param):
    if kind == "sphere":
        return sphere_shape(param)
    if kind in _NAMED:
        return _NAMED[kind](param)
    raise GeometryError(f"unknown shape {kind!r}")


class SurfaceMesh:
    """Nodes, outward normals and Jacobian-folded weights (body.py:74-124)."""

    def __init__(self, nodes, normals, weights, thetas=None, phis=None, patch_grid=None,
                 shape=None, center=(0.0, 0.0, 0.0)):
        self.nodes = np.asarray(nodes, dtype=float)
        self.normals = np.asarray(normals, dtype=float)
        self.weights = np.asarray(weights, dtype=float)
        if self.nodes.shape != self.normals.shape or self.nodes.shape[0] != self.weights.shape[0]:
            raise GeometryError("mesh arrays must agree in length")
        self.thetas, self.phis, self.patch_grid, self.shape = thetas, phis, patch_grid, shape
        self.center = np.asarray(center, dtype=float)
        self.area = float(self.weights.sum())
        if self.area <= 0:
            raise GeometryError("surface must have positive area")
        self.h = math.sqrt(self.area / self.nodes.shape[0])

    @property
    def n_nodes(self):
        return self.nodes.shape[0]

    def has_parametrization(self):
        return self.shape is not None and self.patch_grid is not None

    def refined(self, factor):
        """Same surface with the patch counts multiplied (body.py:108-116)."""
        if not self.has_parametrization():
            raise GeometryError("refinement requires a parametrized mesh")
        nt, nph = self.patch_grid
        return make_surface(self.shape, (nt * factor, nph * factor), center=self.center)

    def surface_point(self, theta, phi):
        R = self.shape[2](theta)
        st = np.sin(theta)
        return self.center + R * np.array([st * np.cos(phi), st * np.sin(phi), np.cos(theta)])

    def radial_bound(self, theta):
        return float(self.shape[2](theta))


def make_surface(shape, resolution, center=(0.0, 0.0, 0.0)):
    """Patchwise Gauss-Legendre mesh of a polar profile R(theta) (body.py:127-184).

    resolution: int n for (n, n) patches or (n_theta, n_phi).  Nodes are
    patch-major, each patch a 4x4 (theta, phi) tensor block.
    """
    if isinstance(shape, tuple) and len(shape) == 2:
        shape = named_shape(*shape)
    kind, param, R, Rp = shape
    nt, nph = (resolution, resolution) if isinstance(resolution, int) else resolution
    if nt < 2 or nph < 2:
        raise GeometryError("need at least 2 patches per direction")
    te = np.linspace(0.0, np.pi, nt + 1)
    pe = np.linspace(0.0, 2.0 * np.pi, nph + 1)
    # per patch (it, ip): theta nodes x phi nodes, theta-major inside the patch
    tn = te[:-1, None] + np.diff(te)[:, None] * GL01_NODES[None, :]      # (nt, 4)
    tw = np.diff(te)[:, None] * GL01_WEIGHTS[None, :]
    pn = pe[:-1, None] + np.diff(pe)[:, None] * GL01_NODES[None, :]      # (nph, 4)
    pw = np.diff(pe)[:, None] * GL01_WEIGHTS[None, :]
    th = np.broadcast_to(tn[:, None, :, None], (nt, nph, 4, 4)).reshape(-1)
    ph = np.broadcast_to(pn[None, :, None, :], (nt, nph, 4, 4)).reshape(-1)
    wp = (tw[:, None, :, None] * pw[None, :, None, :]).reshape(-1)
    r = np.asarray(R(th), dtype=float)
    if np.any(r <= 0):
        raise GeometryError("radius profile must be positive on [0, pi]")
    rp = np.asarray(Rp(th), dtype=float)
    st, ct, sp, cp = np.sin(th), np.cos(th), np.sin(ph), np.cos(ph)
    pos = np.stack([r * st * cp, r * st * sp, r * ct], axis=1)
    drho = rp * st + r * ct
    dz = rp * ct - r * st
    x_t = np.stack([drho * cp, drho * sp, dz], axis=1)
    x_p = np.stack([-r * st * sp, r * st * cp, np.zeros_like(th)], axis=1)
    cr = np.cross(x_t, x_p)
    J = np.linalg.norm(cr, axis=1)
    normals = cr / np.where(J > 0, J, 1.0)[:, None]
    return SurfaceMesh(pos + np.asarray(center, dtype=float), normals, wp * J, thetas=th,
                       phis=ph, patch_grid=(nt, nph), shape=(kind, param, R, Rp), center=center)


def make_icosphere(radius, subdivisions, center=(0.0, 0.0, 0.0)):
    """Icosphere triangle mesh of a sphere (BASELINE config 4 asks for a
    40,962-vertex icosphere: subdivisions = 6 gives 10 * 4^6 + 2 vertices;
    the reference supports only patch meshes, make_surface).  Nodes are the
    vertices projected onto the sphere, normals radial, weights the vertex
    share (1/3) of the adjacent flat triangles' areas, scaled so they sum to
    the sphere's area (vertex quadrature, second order).  The mesh carries
    the sphere's shape (containment and overlap tests) but no patch grid, so
    targets in its near shell cannot get near-surface maps (GeometryError)."""
    if radius <= 0 or subdivisions < 0:
        raise GeometryError("icosphere needs a positive radius and subdivisions >= 0")
    t = (1.0 + math.sqrt(5.0)) / 2.0
    verts = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
             (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    V = np.array(verts, dtype=float)
    V /= np.linalg.norm(V, axis=1)[:, None]
    F = np.array(faces, dtype=np.int64)
    for _ in range(subdivisions):
        # one midpoint per edge, shared by its two faces
        e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
        e.sort(axis=1)
        uniq, inv = np.unique(e, axis=0, return_inverse=True)
        mid = V[uniq[:, 0]] + V[uniq[:, 1]]
        mid /= np.linalg.norm(mid, axis=1)[:, None]
        m = inv.reshape(3, -1) + V.shape[0]          # midpoints of edges 01, 12, 20
        V = np.vstack([V, mid])
        a, b, c = F[:, 0], F[:, 1], F[:, 2]
        F = np.concatenate([np.stack([a, m[0], m[2]], 1), np.stack([b, m[1], m[0]], 1),
                            np.stack([c, m[2], m[1]], 1), np.stack([m[0], m[1], m[2]], 1)])
    r = float(radius)
    P = V * r
    tri = np.cross(P[F[:, 1]] - P[F[:, 0]], P[F[:, 2]] - P[F[:, 0]])
    area = 0.5 * np.linalg.norm(tri, axis=1)
    w = np.zeros(V.shape[0])
    for k in range(3):
        np.add.at(w, F[:, k], area / 3.0)
    w *= 4.0 * math.pi * r * r / w.sum()
    th = np.arccos(np.clip(V[:, 2], -1.0, 1.0))
    ph = np.arctan2(V[:, 1], V[:, 0]) % (2.0 * math.pi)
    mesh = SurfaceMesh(P + np.asarray(center, dtype=float), V.copy(), w, thetas=th, phis=ph,
                       patch_grid=None, shape=sphere_shape(r), center=center)
    mesh.triangles = F
    return mesh


class RigidParticle:
    """Closed rigid surface with its double-layer density and wrenches (body.py:197-215)."""

    def __init__(self, mesh, center=None):
        self._dev = None        # devstate.DeviceState holding the step unknowns
        self.mesh = mesh
        self.center = np.asarray(center if center is not None else mesh.center, dtype=float)
        self.q = np.zeros((mesh.n_nodes, 3))
        self.U = np.zeros(3)
        self.omega = np.zeros(3)
        self.F_ext = np.zeros(3)
        self.L_ext = np.zeros(3)

    # mesh (its nodes), center, q, U and omega live on the device between
    # implicit steps (devstate.DeviceState): reading brings the state back,
    # writing hands it back to the host
    def _get(self, name):
        if self._dev is not None:
            self._dev.pull()
        return self.__dict__["_" + name]

    def _set(self, name, value):
        if self.__dict__.get("_dev") is not None:
            self._dev.release()
        self.__dict__["_" + name] = value

    mesh = property(lambda self: self._get("mesh"), lambda self, v: self._set("mesh", v))
    center = property(lambda self: self._get("center"), lambda self, v: self._set("center", v))
    q = property(lambda self: self._get("q"), lambda self, v: self._set("q", v))
    U = property(lambda self: self._get("U"), lambda self, v: self._set("U", v))
    omega = property(lambda self: self._get("omega"), lambda self, v: self._set("omega", v))

    @property
    def n_nodes(self):
        """Mesh node count (static; never reads the state back)."""
        return self.__dict__["_mesh"].n_nodes

    def translate(self, displacement):
        d = np.asarray(displacement, dtype=float)
        m = self.mesh
        self.mesh = SurfaceMesh(m.nodes + d, m.normals, m.weights, m.thetas, m.phis,
                                m.patch_grid, m.shape, m.center + d)
        self.center = self.center + d


class Periphery:
    """Confining outer surface; fluid on its interior side (body.py:218-234)."""

    def __init__(self, mesh):
        # the reference needs a patch-parametrized mesh; a star-shaped mesh
        # without patches (make_icosphere) is accepted for BASELINE config
        # 4's icosphere -- containment uses its shape, and only near-surface
        # maps need the patches
        if not (mesh.has_parametrization() or (mesh.shape is not None and
                                               getattr(mesh, "triangles", None) is not None)):
            raise GeometryError("periphery requires a parametrized mesh")
        self._dev = None        # devstate.DeviceState holding the density
        self.mesh = mesh
        self.q = np.zeros((mesh.n_nodes, 3))

    @property
    def q(self):
        if self._dev is not None:
            self._dev.pull()
        return self._q

    @q.setter
    def q(self, value):
        if self.__dict__.get("_dev") is not None:
            self._dev.release()
        self._q = value

    def contains(self, points, margin=0.0):
        pts = np.atleast_2d(np.asarray(points, dtype=float)) - self.mesh.center
        rho = np.linalg.norm(pts, axis=1)
        with np.errstate(invalid="ignore"):
            th = np.arccos(np.clip(np.where(rho > 0, pts[:, 2] / np.where(rho > 0, rho, 1.0), 1.0),
                                   -1, 1))
        return rho <= np.asarray(self.mesh.shape[2](th), dtype=float) - margin


# -- per-surface operator API (body.py:237-283, 522-527) on the device --------

def double_layer_offsurface(mesh, q, targets, mu, allow_near=False):
    """Stresslet quadrature at targets away from the surface (body.py:237-251)."""
    from . import kernels
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    q = np.asarray(q, dtype=float)
    if not allow_near:
        d = targets[:, None, :] - mesh.nodes[None, :, :]
        if np.any((d * d).sum(axis=2).min(axis=1) < (NEAR_SHELL_FACTOR * mesh.h) ** 2):
            raise kernels.NearFieldError(
                "target inside the near shell; route through near_surface_eval")
    qw = q * mesh.weights[:, None]
    out, bad = kernels.stresslet_sum(targets, kernels.no_groups(targets.shape[0]), mesh.nodes,
                                     kernels.no_groups(mesh.n_nodes), mesh.normals, qw,
                                     -3.0 / (4.0 * np.pi * mu))
    if bad:
        raise kernels.SingularEvaluationError("target coincides with a mesh node")
    return out


def double_layer_onsurface(mesh, q, mu):
    """Singularity-subtracted on-surface double layer (body.py:254-262)."""
    from . import kernels
    return kernels.stresslet_sum_subtracted(mesh.nodes, mesh.normals, mesh.weights,
                                            np.asarray(q, dtype=float), -3.0 / (4.0 * np.pi * mu))


def completion_flow(particle, targets, mu):
    """Stokeslet + rotlet of the particle's external wrench at its centre
    (body.py:272-283), by the device kernel sf_wrench_flow."""
    import ctypes

    import torch

    from . import _native, kernels
    _native.load(require_device=True)
    targets = np.atleast_2d(np.asarray(targets, dtype=float))
    if np.any(np.linalg.norm(targets - particle.center, axis=1) < kernels.MIN_SEPARATION):
        raise kernels.SingularEvaluationError("target at the particle center")
    f64 = dict(dtype=torch.float64, device="cuda")
    t = torch.as_tensor(targets, **f64).contiguous()
    c = torch.as_tensor(particle.center, **f64)
    w = torch.as_tensor(np.concatenate([particle.F_ext, particle.L_ext]), **f64)
    u = torch.zeros_like(t)
    _native.call("sf_wrench_flow", t.data_ptr(), t.shape[0], c.data_ptr(), w.data_ptr(), float(mu),
                 u.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    return u.cpu().numpy()


def near_surface_eval(mesh, q, target, mu, interior_jump=True, upsample=6):
    """Velocity at a target close to the surface (body.py:522-527): the
    device-built near map (nearfield.device_surface_weights) applied to q."""
    import torch

    from . import nearfield
    Wn = nearfield.device_surface_weights(mesh, np.asarray(target, dtype=float)[None, :], mu,
                                          torch.device("cuda"), interior_jump=interior_jump,
                                          upsample=upsample)[0]
    qd = torch.as_tensor(np.asarray(q, dtype=float).ravel(), dtype=torch.float64, device="cuda")
    corr = (Wn @ qd).cpu().numpy()                       # (W_near - W_plain) q
    plain = double_layer_offsurface(mesh, q, np.asarray(target, dtype=float)[None, :], mu,
                                    allow_near=True)[0]  # W_plain q
    return plain + corr


# -- small host helpers (body.py:186-193, 265-295) ---------------------------

def surface_integral(mesh, f):
    """Quadrature sum of scalar or vector nodal data."""
    f = np.asarray(f, dtype=float)
    if f.shape[0] != mesh.n_nodes:
        raise ValueError("nodal data does not conform to the mesh")
    return float(mesh.weights @ f) if f.ndim == 1 else mesh.weights @ f


def nullspace_operator(periphery, q):
    """n(x) times the flux of q through the periphery."""
    mesh = periphery.mesh if isinstance(periphery, Periphery) else periphery
    flux = float(mesh.weights @ (mesh.normals * np.asarray(q, dtype=float)).sum(axis=1))
    return mesh.normals * flux


def rigid_constraint_averages(particle, q):
    """Area averages of q and of its moment about the centre."""
    mesh = particle.mesh
    if mesh.area <= 0:
        raise GeometryError("zero-area surface")
    q = np.asarray(q, dtype=float)
    wq = mesh.weights[:, None] * q
    return wq.sum(axis=0) / mesh.area, \
        (mesh.weights[:, None] * np.cross(mesh.nodes - particle.center, q)).sum(axis=0) / mesh.area


# -- nodal interpolation and nearly singular helpers (body.py:305-519) --------

def _lagrange_coeffs(x, nodes):
    x = np.atleast_1d(np.asarray(x, dtype=float))
    c = np.ones((x.size, len(nodes)))
    for i in range(len(nodes)):
        for j in range(len(nodes)):
            if i != j:
                c[:, i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return c


def _patch_coeffs(mesh, theta, phi):
    nt, nph = mesh.patch_grid
    dth, dph = np.pi / nt, 2.0 * np.pi / nph
    it = np.minimum((theta / dth).astype(int), nt - 1)
    ip = np.minimum((phi / dph).astype(int), nph - 1)
    return (it * nph + ip, _lagrange_coeffs((theta - it * dth) / dth, GL01_NODES),
            _lagrange_coeffs((phi - ip * dph) / dph, GL01_NODES))


def interpolate_nodal(mesh, values, theta, phi):
    """Nodal data at (theta, phi) by 4x4 tensor Lagrange interpolation in the
    containing patch (body.py:316-338)."""
    if not mesh.has_parametrization():
        raise GeometryError("interpolation requires a parametrized mesh")
    scalar_query = np.isscalar(theta)
    theta = np.atleast_1d(np.asarray(theta, dtype=float))
    phi = np.atleast_1d(np.asarray(phi, dtype=float)) % (2.0 * np.pi)
    patch, cu, cv = _patch_coeffs(mesh, theta, phi)
    vals = np.asarray(values, dtype=float)
    flat = vals.reshape(vals.shape[0], -1)
    block = flat[(patch * 16)[:, None] + np.arange(16)].reshape(theta.size, 4, 4, -1)
    out = np.einsum("mi,mj,mijk->mk", cu, cv, block)
    if vals.ndim == 1:
        out = out[:, 0]
    return (out[0] if vals.ndim > 1 else float(out[0])) if scalar_query else out


def interpolation_matrix(mesh, fine):
    """Sparse nodal map mesh -> fine reproducing interpolate_nodal at the
    fine nodes (body.py:341-368)."""
    from scipy import sparse
    if not mesh.has_parametrization():
        raise GeometryError("interpolation requires a parametrized mesh")
    theta = np.asarray(fine.thetas, dtype=float)
    phi = np.asarray(fine.phis, dtype=float) % (2.0 * np.pi)
    patch, cu, cv = _patch_coeffs(mesh, theta, phi)
    vals = np.einsum("mi,mj->mij", cu, cv).reshape(theta.size, 16)
    cols = (patch * 16)[:, None] + np.arange(16)
    rows = np.repeat(np.arange(theta.size), 16)
    return sparse.csr_matrix((vals.ravel(), (rows, cols.ravel())),
                             shape=(theta.size, mesh.n_nodes))


def _plain_surface_map_device(mesh, targets, mu, dev):
    """The stresslet quadrature map (k, 3, 3N) at k targets (body.py:437-448)
    on the device: block j = -3/(4 pi mu) w_j (r.n_j) r r^T / r^5, r = t - y_j."""
    import torch
    f64 = dict(dtype=torch.float64, device=dev)
    t = torch.as_tensor(np.atleast_2d(targets), **f64)
    y = torch.as_tensor(mesh.nodes, **f64)
    nrm = torch.as_tensor(mesh.normals, **f64)
    w = torch.as_tensor(mesh.weights, **f64)
    r = t[:, None, :] - y[None, :, :]
    d2 = (r * r).sum(dim=2)
    s = (-3.0 / (4.0 * np.pi * mu)) * w[None, :] * (r * nrm[None, :, :]).sum(dim=2) / (
        d2 * d2 * torch.sqrt(d2))
    blocks = s[..., None, None] * r[..., :, None] * r[..., None, :]
    return blocks.permute(0, 2, 1, 3).reshape(t.shape[0], 3, -1)


def plain_surface_weights(mesh, target, mu):
    """Stresslet quadrature at one target as a (3, 3N) map (body.py:437-448),
    evaluated on the device."""
    import torch
    return _plain_surface_map_device(mesh, target, mu, torch.device("cuda"))[0].cpu().numpy()


def near_surface_weights(mesh, target, mu, interior_jump=True, upsample=6):
    """Nearly singular (3, 3N) map (body.py:479-519), built on the device
    (nearfield.device_surface_weights returns W_near - W_plain; the plain
    map is added back on the device)."""
    import torch

    from . import nearfield
    dev = torch.device("cuda")
    t = np.asarray(target, dtype=float)[None, :]
    W = nearfield.device_surface_weights(mesh, t, mu, dev, interior_jump=interior_jump,
                                         upsample=upsample)[0]
    return (W + _plain_surface_map_device(mesh, t, mu, dev)[0]).cpu().numpy()


def second_kind_matrix(mesh, mu, interior=True, nullspace_scale=None):
    """Dense one-sided double-layer matrix (body.py:530-566) for small
    meshes, assembled on the device."""
    import torch
    dev = torch.device("cuda")
    f64 = dict(dtype=torch.float64, device=dev)
    x = torch.as_tensor(mesh.nodes, **f64)
    n = torch.as_tensor(mesh.normals, **f64)
    w = torch.as_tensor(mesh.weights, **f64)
    N = mesh.n_nodes
    pref = -3.0 / (4.0 * np.pi * mu)
    r = x[:, None, :] - x[None, :, :]
    d2 = (r * r).sum(dim=2)
    d2.fill_diagonal_(1.0)
    rhat = r / torch.sqrt(d2)[:, :, None]
    scal = pref * (rhat * n[None, :, :]).sum(dim=2) / d2 * w[None, :]
    blocks = scal[:, :, None, None] * rhat[:, :, None, :] * rhat[:, :, :, None]
    idx = torch.arange(N, device=dev)
    blocks[idx, idx] = 0.0
    A = blocks.permute(0, 2, 1, 3).reshape(3 * N, 3 * N).clone()
    rowsum = blocks.sum(dim=1)
    for i in range(N):
        A[3 * i:3 * i + 3, 3 * i:3 * i + 3] -= rowsum[i]
    if interior:
        A += torch.eye(3 * N, **f64) / mu
    if nullspace_scale is not None:
        nw = (n * w[:, None]).reshape(-1)
        A += nullspace_scale * torch.outer(n.reshape(-1), nw)
    return A.cpu().numpy()
