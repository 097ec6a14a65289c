"""The implicit step's state resident on the device between steps.

The reference keeps every constituent's unknowns in host arrays and writes
them back after each solve (solver.py:558-573: q, U, omega, the particle
translation, X, T, refresh_geometry).  Here the step writes them into a
DeviceState instead: per Chebyshev order class the centrelines X (nb, n, 3)
and tensions T (nb, n); per rigid particle its mesh nodes, centre, U, omega
and density q; the periphery density.  The next step's InteractionCache and
BlockOperator read them directly (geometry refreshed by
sf_fiber_geometry_batched from these tensors), so a run of steps moves no
state through the host.

The host objects (fiber.Fiber, body.RigidParticle, body.Periphery) keep
their attributes: reading one brings the whole state back in one transfer
(`pull`), writing one hands the state back to the host (`release`: the next
step uploads it again).  So user code that inspects or edits a state between
steps sees exactly the reference's values.
"""

import numpy as np


class DeviceState:
    def __init__(self, state, device):
        import torch

        from .system import order_classes
        self.device = device
        f64 = dict(dtype=torch.float64, device=device)
        self.fibers = list(state.fibers)
        self.particles = list(state.particles)
        self.periphery = state.periphery
        self.classes = []
        for n, idx in order_classes(self.fibers):
            X = np.stack([self.fibers[m]._X for m in idx])
            T = np.stack([self.fibers[m]._T for m in idx])
            self.classes.append((n, idx, torch.as_tensor(X, **f64), torch.as_tensor(T, **f64)))
        self.pnodes, self.pnrm, self.pw, self.pq = [], [], [], []
        for part in self.particles:
            m = part.__dict__["_mesh"]
            self.pnodes.append(torch.as_tensor(m.nodes, **f64))
            self.pnrm.append(torch.as_tensor(m.normals, **f64))
            self.pw.append(torch.as_tensor(m.weights, **f64))
            self.pq.append(torch.as_tensor(np.asarray(part.__dict__["_q"], dtype=float)
                                           .reshape(-1, 3), **f64))
        npart = len(self.particles)
        if npart:
            self.pcenter = torch.as_tensor(np.stack([p.__dict__["_center"] for p in self.particles]),
                                           **f64)
            self.pU = torch.as_tensor(np.stack([p.__dict__["_U"] for p in self.particles]), **f64)
            self.pomega = torch.as_tensor(np.stack([p.__dict__["_omega"] for p in self.particles]),
                                          **f64)
            self.pmesh_center = torch.as_tensor(
                np.stack([p.__dict__["_mesh"].center for p in self.particles]), **f64)
        else:
            self.pcenter = self.pU = self.pomega = self.pmesh_center = None
        self.q0 = None
        if self.periphery is not None:
            per = self.periphery
            self.q0 = torch.as_tensor(np.asarray(per._q, dtype=float).reshape(-1, 3), **f64)
            m = per.mesh
            self.per_nodes = torch.as_tensor(m.nodes, **f64)
            self.per_nrm = torch.as_tensor(m.normals, **f64)
            self.per_w = torch.as_tensor(m.weights, **f64)
        self._gather = None
        self.stale = False          # host copies older than the device
        self.alive = True
        for obj in self._objects():
            obj._dev = self

    def _objects(self):
        out = list(self.fibers) + list(self.particles)
        if self.periphery is not None:
            out.append(self.periphery)
        return out

    # -- host synchronisation -------------------------------------------------
    def pull(self):
        """Copy the device state into the host objects (once per stale
        period; one transfer per array family)."""
        if not self.stale or not self.alive:
            return
        self.stale = False
        from .body import SurfaceMesh
        for n, idx, X, T in self.classes:
            Xh, Th = X.cpu().numpy(), T.cpu().numpy()
            for k, m in enumerate(idx):
                f = self.fibers[m]
                f._X = Xh[k].copy()
                f._T = Th[k].copy()
                f._geo = None
        if self.particles:
            cen = self.pcenter.cpu().numpy()
            U = self.pU.cpu().numpy()
            om = self.pomega.cpu().numpy()
            mc = self.pmesh_center.cpu().numpy()
            for i, part in enumerate(self.particles):
                d = part.__dict__
                m = d["_mesh"]
                d["_mesh"] = SurfaceMesh(self.pnodes[i].cpu().numpy(), m.normals, m.weights,
                                         m.thetas, m.phis, m.patch_grid, m.shape, mc[i].copy())
                d["_center"] = cen[i].copy()
                d["_U"] = U[i].copy()
                d["_omega"] = om[i].copy()
                d["_q"] = self.pq[i].cpu().numpy().copy()
        if self.periphery is not None:
            self.periphery._q = self.q0.cpu().numpy().copy()

    def release(self):
        """Hand the state back to the host for good (a host write is about
        to happen): pull, then detach from every object."""
        if not self.alive:
            return
        self.pull()
        self.alive = False
        for obj in self._objects():
            if obj.__dict__.get("_dev") is self:
                obj._dev = None

    def matches(self, state):
        """True while this mirror still describes `state` (same constituents,
        no host write since)."""
        if not self.alive or len(state.fibers) != len(self.fibers) or \
                len(state.particles) != len(self.particles) or state.periphery is not self.periphery:
            return False
        return all(a is b for a, b in zip(state.fibers, self.fibers)) and \
            all(a is b for a, b in zip(state.particles, self.particles))

    # -- the step's write-back (solver.py:558-573) -----------------------------
    def _indices(self, layout):
        import torch
        if self._gather is None:
            dev = self.device
            g = []
            for n, idx, _, _ in self.classes:
                xs = np.concatenate([np.arange(layout.X[m].start, layout.X[m].stop) for m in idx])
                ts = np.concatenate([np.arange(layout.T[m].start, layout.T[m].stop) for m in idx])
                g.append((torch.as_tensor(xs, device=dev), torch.as_tensor(ts, device=dev)))
            self._gather = g
        return self._gather

    def write_solution(self, sol, layout, dt):
        """X, T, U, omega, q1, q0 from the solved unknowns; particles translate
        by dt U (mesh nodes, mesh centre and centre, as RigidParticle.translate).
        New tensors, so caches of the finished step keep their geometry."""
        for c, (xi, ti) in enumerate(self._indices(layout)):
            n, idx, _, _ = self.classes[c]
            self.classes[c] = (n, idx, sol[xi].view(idx.size, n, 3), sol[ti].view(idx.size, n))
        if self.particles:
            import torch
            U = torch.stack([sol[s] for s in layout.U])
            self.pU = U
            self.pomega = torch.stack([sol[s] for s in layout.omega])
            d = dt * U
            self.pq = [sol[s].view(-1, 3).clone() for s in layout.q1]
            self.pnodes = [self.pnodes[i] + d[i] for i in range(len(self.particles))]
            self.pmesh_center = self.pmesh_center + d
            self.pcenter = self.pcenter + d
        if self.periphery is not None:
            self.q0 = sol[layout.q0].view(-1, 3).clone()
        self.stale = True

    def fiber_X(self):
        """[(n, idx, X (nb, n, 3))] per order class."""
        return [(n, idx, X) for n, idx, X, _ in self.classes]

    def unknowns_vector(self, layout):
        """The current state packed as step unknowns (solver.warm_start_vector)."""
        import torch
        x0 = torch.zeros(layout.size, dtype=torch.float64, device=self.device)
        for c, (xi, ti) in enumerate(self._indices(layout)):
            _, _, X, T = self.classes[c]
            x0[xi] = X.reshape(-1)
            x0[ti] = T.reshape(-1)
        for i in range(len(self.particles)):
            x0[layout.U[i]] = self.pU[i]
            x0[layout.omega[i]] = self.pomega[i]
            x0[layout.q1[i]] = self.pq[i].reshape(-1)
        if self.periphery is not None:
            x0[layout.q0] = self.q0.reshape(-1)
        return x0


def for_state(state, device):
    """The state's device mirror, built (uploaded) when missing or stale."""
    dev = getattr(state, "_dev", None)
    if dev is not None and dev.matches(state) and dev.device == device:
        return dev
    if dev is not None:
        dev.release()
    for obj in list(state.fibers) + list(state.particles) + (
            [state.periphery] if state.periphery is not None else []):
        other = obj.__dict__.get("_dev")
        if other is not None:
            other.release()
    dev = DeviceState(state, device)
    state._dev = dev
    return dev


def mirror_of(state):
    """The state's live device mirror, or None."""
    dev = getattr(state, "_dev", None)
    return dev if dev is not None and dev.matches(state) else None
