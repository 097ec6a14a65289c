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


def make_surface(shape, resolution, center=(0.0, 0.0, 0.0)):
    """Patchwise Gauss-Legendre mesh of a polar profile R(theta) (body.py:127-184).

    resolution: int n for (n, n) patches or (n_theta, n_phi).  Nodes are
    patch-major, each patch a 4x4 (theta, phi) tensor block.
    """
    if isinstance(shape, tuple) and len(shape) == 2:
        if shape[0] != "sphere":
            raise GeometryError(f"unknown shape {shape[0]!r}")
        shape = sphere_shape(shape[1])
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


class RigidParticle:
    """Closed rigid surface with its double-layer density and wrenches (body.py:197-215)."""

    def __init__(self, mesh, center=None):
        self.mesh = mesh
        self.center = np.asarray(center if center is not None else mesh.center, dtype=float)
        self.q = np.zeros((mesh.n_nodes, 3))
        self.U = np.zeros(3)
        self.omega = np.zeros(3)
        self.F_ext = np.zeros(3)
        self.L_ext = np.zeros(3)

    def translate(self, displacement):
        d = np.asarray(displacement, dtype=float)
        m = self.mesh
        self.mesh = SurfaceMesh(m.nodes + d, m.normals, m.weights, m.thetas, m.phis,
                                m.patch_grid, m.shape, m.center + d)
        self.center = self.center + d


class Periphery:
    """Confining outer surface; fluid on its interior side (body.py:218-234)."""

    def __init__(self, mesh):
        if not mesh.has_parametrization():
            raise GeometryError("periphery requires a parametrized mesh")
        self.mesh = mesh
        self.q = np.zeros((mesh.n_nodes, 3))

    def contains(self, points, margin=0.0):
        pts = np.atleast_2d(np.asarray(points, dtype=float)) - self.mesh.center
        rho = np.linalg.norm(pts, axis=1)
        with np.errstate(invalid="ignore"):
            th = np.arccos(np.clip(np.where(rho > 0, pts[:, 2] / np.where(rho > 0, rho, 1.0), 1.0),
                                   -1, 1))
        return rho <= np.asarray(self.mesh.shape[2](th), dtype=float) - margin
