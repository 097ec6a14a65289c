"""Generate golden vectors by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Imports `slenderflow` read-only from /root/reference/pkg/src and stores its
outputs on seeded inputs as small .npz fixtures next to this script.  The
fixtures travel with the repo; nothing at test time reads /root/reference.
Inputs (fiber centrelines) come from paper_1602_05650_b200.configs so the
device path, the oracle and the reference see bit-identical arrays.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import numba  # noqa: E402
import scipy  # noqa: E402
from slenderflow import body, fiber, kernels, system  # noqa: E402

from paper_1602_05650_b200 import configs  # noqa: E402


def versions():
    return dict(numpy=np.__version__, scipy=scipy.__version__, numba=numba.__version__)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def pairs_small():
    """Pair kernels on random inputs, with group exclusion and coincidences."""
    rng = np.random.default_rng(2024)
    ns, nt = 300, 200
    src = rng.standard_normal((ns, 3)) * 1.5
    sgrp = np.repeat(np.arange(10, dtype=np.int64), 30)
    f = rng.standard_normal((ns, 3))
    trg = rng.standard_normal((nt, 3)) * 1.5
    tgrp = rng.integers(-1, 10, nt).astype(np.int64)
    # coincidences: target 0 on source 5 (same group -> excluded, not bad);
    # target 1 on source 40 in a different group -> bad
    trg[0] = src[5]
    tgrp[0] = sgrp[5]
    trg[1] = src[40]
    tgrp[1] = 7
    pref = 1.0 / (8.0 * np.pi * 0.9)
    st, st_bad = kernels.stokeslet_sum(trg, tgrp, src, sgrp, f, pref)
    db, db_bad = kernels.doublet_sum(trg, tgrp, src, sgrp, f, pref)
    nrm = rng.standard_normal((ns, 3))
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    qw = rng.standard_normal((ns, 3))
    sp = -3.0 / (4.0 * np.pi * 1.1)
    ss, ss_bad = kernels.stresslet_sum(trg, tgrp, src, sgrp, nrm, qw, sp)
    # surface self terms on a sphere mesh
    mesh = body.make_surface(body.sphere_shape(1.3), (4, 6))
    q = rng.standard_normal((mesh.n_nodes, 3))
    sub = kernels.stresslet_sum_subtracted(mesh.nodes, mesh.normals, mesh.weights, q, sp)
    rsum = kernels.stresslet_rowsum(mesh.nodes, mesh.normals, mesh.weights, sp)
    const = np.tile([0.4, -1.0, 2.0], (mesh.n_nodes, 1))
    sub_const = kernels.stresslet_sum_subtracted(mesh.nodes, mesh.normals, mesh.weights, const, sp)
    # K_delta of a bent fiber
    p = 24
    g = fiber.shared_grid(p)
    th = (g.nodes + 1.0) * 0.4
    X = np.stack([np.cos(th), np.sin(th), 0.1 * th], axis=1)
    fib = fiber.Fiber(X, eps=0.01, E=1.0)
    K = fib.kdelta_matrix(0.7)
    save("pairs_small.npz", src=src, sgrp=sgrp, f=f, trg=trg, tgrp=tgrp, pref=pref,
         stokeslet=st, stokeslet_bad=st_bad, doublet=db, doublet_bad=db_bad,
         nrm=nrm, qw=qw, spref=sp, stresslet=ss, stresslet_bad=ss_bad,
         mesh_nodes=mesh.nodes, mesh_normals=mesh.normals, mesh_weights=mesh.weights,
         q=q, subtracted=sub, rowsum=rsum, subtracted_const=sub_const,
         kd_X=X, kd_s=fib.s, kd_sa=fib.s_alpha, kd_t=fib.tangents, kd_w=g.weights,
         kd_delta=fib.delta, kd_pref=1.0 / (8.0 * np.pi * 0.7), kd_K=K, **versions())


def operator_fixture(name, cloud, seed_f=1, mu=1.0, keep_k=2):
    """C1-form HI operator: complementary_velocities + local self terms."""
    f = configs.forces(cloud, seed=seed_f)
    fibs = [fiber.Fiber(X, eps=cloud.eps, E=cloud.E) for X in cloud.X]
    st = system.SystemState(fibs, mu=mu)
    cache = system.InteractionCache(st)
    res = system.complementary_velocities(st, fiber_forces=list(f), cache=cache)
    u_nl = np.vstack(res.fibers)
    u_self = np.vstack([fiber.local_mobility_apply(fb, fm, mu) + fiber.nonlocal_Kdelta_apply(fb, fm, mu)
                        for fb, fm in zip(fibs, f)])
    near_t = np.array([t for t, _, _ in cache.near_fiber], dtype=np.int64)
    near_l = np.array([l for _, l, _ in cache.near_fiber], dtype=np.int64)
    near_W = (np.stack([W for _, _, W in cache.near_fiber]) if cache.near_fiber
              else np.zeros((0, 3, 3 * cloud.n_nodes)))
    geo = dict(s=np.stack([fb.s for fb in fibs]), s_alpha=np.stack([fb.s_alpha for fb in fibs]),
               tangents=np.stack([fb.tangents for fb in fibs]), L=np.array([fb.L for fb in fibs]),
               delta=np.array([fb.delta for fb in fibs]),
               weights=np.stack([fb.node_weights() for fb in fibs]))
    Ks = np.stack([fibs[m].kdelta_matrix(mu) for m in range(keep_k)])
    save(name, X=cloud.X, forces=f, eps=cloud.eps, E=cloud.E, mu=mu, p=cloud.p,
         u_nl=u_nl, u_self=u_self, near_t=near_t, near_l=near_l, near_W=near_W, K=Ks,
         **geo, **versions())
    print(f"  {name}: {len(cache.near_fiber)} near pairs")


def surfaces_fixture():
    """Fibers + rigid particle + periphery: every surface term of the operator."""
    per = body.Periphery(body.make_surface(body.sphere_shape(6.0), (8, 8)))
    part = body.RigidParticle(body.make_surface(body.sphere_shape(1.0), (6, 6)))
    part.F_ext = np.array([0.3, -0.1, 2.0])
    part.L_ext = np.array([0.05, 0.2, -0.1])
    fibs = [fiber.straight_fiber(15, (2.5, 0.0, -1.0), (0, 0, 1.0), 2.0),
            fiber.straight_fiber(15, (-2.4, 0.5, -0.5), (0.6, 0.8, 0.0), 1.5),
            fiber.straight_fiber(15, (0.3, 2.6, 0.2), (0.0, 0.6, 0.8), 1.8)]
    st = system.SystemState(fibs, [part], per)
    rng = np.random.default_rng(99)
    q0 = rng.standard_normal((per.mesh.n_nodes, 3)) * 0.1
    q1 = rng.standard_normal((part.mesh.n_nodes, 3)) * 0.1
    f = [rng.standard_normal((16, 3)) for _ in fibs]
    wrench = (part.F_ext, part.L_ext)
    cache = system.InteractionCache(st)
    res = system.complementary_velocities(st, periphery_density=q0, particle_densities=[q1],
                                          fiber_forces=f, particle_wrenches=[wrench], cache=cache)
    mu = st.mu
    save("surfaces.npz",
         per_nodes=per.mesh.nodes, per_normals=per.mesh.normals, per_weights=per.mesh.weights,
         part_nodes=part.mesh.nodes, part_normals=part.mesh.normals,
         part_weights=part.mesh.weights, part_center=part.center,
         F_ext=part.F_ext, L_ext=part.L_ext,
         X=np.stack([fb.X for fb in fibs]), eps=0.01, L=np.array([fb.L for fb in fibs]),
         weights=np.stack([fb.node_weights() for fb in fibs]), forces=np.stack(f),
         q0=q0, q1=q1, u_per=res.periphery, u_part=res.particles[0],
         u_fib=np.vstack(res.fibers), n_near_fiber=len(cache.near_fiber),
         n_near_surface=len(cache.near_surface),
         dl_on_per=body.double_layer_onsurface(per.mesh, q0, mu),
         dl_on_part=body.double_layer_onsurface(part.mesh, q1, mu),
         rowsum_part=kernels.stresslet_rowsum(part.mesh.nodes, part.mesh.normals,
                                              part.mesh.weights, -3.0 / (4.0 * np.pi * mu)),
         **versions())
    print(f"  surfaces: near fiber {len(cache.near_fiber)}, near surface {len(cache.near_surface)}")


# ---------------------------------------------------------------- implicit steps
def _step_record(state):
    ragged = len({f.n_nodes for f in state.fibers}) > 1
    cat = np.concatenate if ragged else np.stack
    return dict(X=cat([f.X for f in state.fibers]), T=cat([f.T for f in state.fibers]),
                U=np.stack([p.U for p in state.particles]) if state.particles else np.zeros((0, 3)),
                omega=(np.stack([p.omega for p in state.particles]) if state.particles
                       else np.zeros((0, 3))),
                q1=(np.stack([p.q for p in state.particles]) if state.particles
                    else np.zeros((0, 1, 3))),
                q0=state.periphery.q if state.periphery is not None else np.zeros((0, 3)))


def aster_state(n_fibers=12, p=15, mesh_res=(4, 4), E=1.0, periphery=False, hinged=False):
    from slenderflow import system as S
    pnc = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), mesh_res))
    pts, dirs = S.aster_attachment_layout(pnc, n_fibers, radius_factor=1.3)
    fibs = []
    for k, (x0, d) in enumerate(zip(pts, dirs)):
        fb = fiber.straight_fiber(p, x0, d, 1.0, eps=1e-2, E=E)
        fb.bc_minus = fiber.ClampedToBody(0, x0, d)
        fb.bc_plus = fiber.PrescribedForceTorque(1.0 * d)
        if hinged and k == 0:
            fb.bc_plus = fiber.HingedToSurface(attachment=fb.X[0] + 0.05 * d, stiffness=10.0)
        fibs.append(fb)
    per = body.Periphery(body.make_surface(body.sphere_shape(3.0), (6, 6))) if periphery else None
    return S.SystemState(fibs, [pnc], per)


def cloud_state(n_fibers=8, p=15, seed=3):
    from slenderflow import system as S
    cl = configs.fiber_cloud(n_fibers, p, eps=5e-3, E=1e-2, region="ball", size=1.5, seed=seed,
                             clear=configs.clean_clear(p), check="node", perturb=1e-2)
    fibs = [fiber.Fiber(X, eps=5e-3, E=1e-2) for X in cl.X]
    return S.SystemState(fibs, force_models=[S.UniformBodyForce(1.0, (0.0, 0.0, -1.0))]), cl.X


def step_fixture(name, state, dt, tol, nsteps, extra=None):
    from slenderflow import solver as R
    rng = np.random.default_rng(5)
    op, rhs = R.assemble_step_operator(state, dt)
    prec = R.Preconditioner(op)
    u = rng.standard_normal(op.layout.size)
    v = rng.standard_normal(op.layout.size)
    rec = dict(apply_u=u, apply_Au=op.apply(u), rhs=rhs, prec_v=v, prec_Mv=prec.apply(v),
               block0=op.fiber_blocks[0], layout_size=op.layout.size)
    init = _step_record(state)
    steps = []
    for _ in range(nsteps):
        params = R.GmresParams(tolerance=tol)
        # iterations of the reference's own solve for the record
        op2, rhs2 = R.assemble_step_operator(state, dt)
        _, iters, hist = R.gmres_solve(op2, R.Preconditioner(op2), rhs2, params)
        R.backward_euler_step(state, dt, params)
        steps.append((iters, _step_record(state)))
    out = dict(dt=dt, tol=tol, nsteps=nsteps, **{f"init_{k}": v for k, v in init.items()}, **rec)
    for s_i, (iters, r) in enumerate(steps):
        out[f"iters_{s_i}"] = iters
        for k, v in r.items():
            out[f"step{s_i}_{k}"] = v
    if extra:
        out.update(extra)
    save(name, **out, **versions())


def mixed_cloud_state():
    """Free fibers of two Chebyshev orders (p = 15 and 23), interleaved."""
    from slenderflow import system as S
    a = configs.fiber_cloud(4, 15, eps=5e-3, E=1e-2, region="ball", size=1.2, seed=3,
                            clear=configs.clean_clear(15), check="node", perturb=1e-2)
    b = configs.fiber_cloud(4, 23, eps=5e-3, E=1e-2, region="ball", size=1.2, seed=4,
                            clear=configs.clean_clear(23), check="node", perturb=1e-2)
    Xs = []
    for k in range(4):
        Xs.append(a.X[k])
        Xs.append(b.X[k] + np.array([3.5, 0.0, 0.0]))
    fibs = [fiber.Fiber(X, eps=5e-3, E=1e-2) for X in Xs]
    return S.SystemState(fibs, force_models=[S.UniformBodyForce(1.0, (0.0, 0.0, -1.0))]), Xs


def mixed_aster_state(n_fibers=10):
    """Aster whose clamped fibers alternate between p = 15 and p = 23."""
    from slenderflow import system as S
    pnc = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4)))
    pts, dirs = S.aster_attachment_layout(pnc, n_fibers, radius_factor=1.3)
    fibs = []
    for k, (x0, d) in enumerate(zip(pts, dirs)):
        fb = fiber.straight_fiber(15 if k % 2 == 0 else 23, x0, d, 1.0, eps=1e-2, E=1.0)
        fb.bc_minus = fiber.ClampedToBody(0, x0, d)
        fb.bc_plus = fiber.PrescribedForceTorque(1.0 * d)
        fibs.append(fb)
    return S.SystemState(fibs, [pnc])


def steps_mixed():
    st, Xs = mixed_cloud_state()
    step_fixture("step_mixed_cloud.npz", st, 5e-3, 1e-10, 2,
                 extra={f"init_X{k}": X for k, X in enumerate(Xs)})
    st = mixed_aster_state()
    step_fixture("step_mixed_aster.npz", st, 1e-3, 1e-10, 2,
                 extra={f"fiber_p": np.array([f.p for f in st.fibers])})


def steps_all():
    st = aster_state()
    step_fixture("step_aster.npz", st, 1e-3, 1e-10, 2)
    st, X0 = cloud_state()
    step_fixture("step_cloud.npz", st, 5e-3, 1e-10, 2, extra=dict(cloud_X=X0))
    st = aster_state(n_fibers=6, periphery=True, hinged=True)
    step_fixture("step_confined.npz", st, 1e-3, 1e-10, 1)


def near_surface_fixture():
    """Near-surface correction maps (body.py:479-519) for a few targets."""
    part = body.make_surface(body.sphere_shape(0.5), (4, 4))
    per = body.make_surface(body.sphere_shape(3.0), (6, 6))
    tp = np.array([[0.0, 0.0, 0.62], [0.3, 0.35, 0.2], [0.5, 0.05, 0.0]])
    tq = np.array([[0.0, 0.0, 2.7], [1.9, 1.9, 0.9], [0.1, -2.85, 0.3]])
    Wp = np.stack([body.near_surface_weights(part, t, 1.0, interior_jump=False)
                   - body.plain_surface_weights(part, t, 1.0) for t in tp])
    Wq = np.stack([body.near_surface_weights(per, t, 1.0, interior_jump=True)
                   - body.plain_surface_weights(per, t, 1.0) for t in tq])
    nsp = [body.nearest_surface_point(per, t) for t in tq]
    save("near_surface.npz", tp=tp, tq=tq, Wp=Wp, Wq=Wq,
         nsp=np.array([[a, b, *x, d] for a, b, x, d in nsp]), **versions())


def bc_fixture(fib, Xc, Tc, mu):
    """bc_residuals (fiber.py:375-441) for every boundary-condition kind."""
    out = {}
    d = fib.tangents[-1]
    kin = dict(U=np.array([0.1, -0.2, 0.05]), omega=np.array([0.3, 0.1, -0.2]),
               center=fib.X[-1] - 0.4 * d, dt=1e-3)
    cases = {
        "free": (fiber.FreeEnd(), fiber.FreeEnd()),
        "pft": (fiber.PrescribedForceTorque([0.5, -1.0, 0.2], [0.1, 0.0, -0.3]), fiber.FreeEnd()),
        "hinged": (fiber.HingedToSurface(fib.X[0] + 0.01, 3.0), fiber.FreeEnd()),
        "clamped": (fiber.FreeEnd(), fiber.ClampedToBody(0, fib.X[-1], d)),
        "clamped_h": (fiber.FreeEnd(), fiber.ClampedToBody(0, fib.X[-1])),
    }
    for name, (bp, bm) in cases.items():
        fib.bc_plus, fib.bc_minus = bp, bm
        for hom in (False, True):
            out[f"bc_{name}_{int(hom)}"] = fiber.bc_residuals(
                fib, Xc, Tc, body_kinematics=kin, mu=mu, u_bar=np.array([0.01, 0.02, -0.03]),
                homogeneous=hom)
    fib.bc_plus, fib.bc_minus = fiber.FreeEnd(), fiber.FreeEnd()
    return out


def api_ops_fixture():
    """Per-constituent operator API of the reference (fiber.py:237-289,
    body.py:237-283, 522-527) on seeded inputs: the functions a reference
    user calls directly."""
    rng = np.random.default_rng(11)
    cl = configs.make("c1_clean", seed=0)
    fib = fiber.Fiber(cl.X[3], eps=1e-2, E=0.7)
    f = rng.standard_normal((fib.n_nodes, 3))
    Xc = cl.X[3] + 1e-3 * rng.standard_normal(cl.X[3].shape)
    Tc = rng.standard_normal(fib.n_nodes)
    mu = 1.3
    far = cl.X[3].mean(axis=0) + np.array([[2.0, 0.5, -1.0], [-1.5, 2.5, 0.3], [0.2, -0.1, 3.0]])
    part = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4)))
    part.F_ext = np.array([0.3, -1.0, 0.5])
    part.L_ext = np.array([-0.2, 0.1, 0.7])
    per = body.make_surface(body.sphere_shape(3.0), (6, 6))
    q = rng.standard_normal((per.n_nodes, 3))
    qp = rng.standard_normal((part.mesh.n_nodes, 3))
    tgt = np.array([[0.1, 0.2, 0.3], [1.0, -0.5, 0.4], [-0.7, 0.6, -1.1]])
    near_t = np.array([0.1, -2.85, 0.3])
    save("api_ops.npz", X=cl.X[3], eps=1e-2, E=0.7, mu=mu, f=f, Xc=Xc, Tc=Tc, far=far,
         elastic=fiber.elastic_force_density(fib, Xc, Tc),
         mobility=fiber.local_mobility_apply(fib, f, mu),
         kdelta=fiber.nonlocal_Kdelta_apply(fib, f, mu),
         induced=fiber.fiber_induced_velocity(fib, f, far, mu),
         induced_dbl=fiber.fiber_induced_velocity(fib, f, far, mu, include_doublet=True),
         q=q, qp=qp, tgt=tgt, near_t=near_t, F=part.F_ext, L=part.L_ext,
         dl_off=body.double_layer_offsurface(per, q, tgt, mu),
         dl_on=body.double_layer_onsurface(per, q, mu),
         dl_on_p=body.double_layer_onsurface(part.mesh, qp, mu),
         completion=body.completion_flow(part, tgt + 1.0, mu),
         near_eval=body.near_surface_eval(per, q, near_t, mu, interior_jump=True),
         Ds4=fib.Ds4, FX=fib.elastic_operators()[0], FT=fib.elastic_operators()[1],
         skm=body.second_kind_matrix(body.make_surface(body.sphere_shape(0.5), (2, 2)), mu,
                                     interior=False),
         skm_per=body.second_kind_matrix(body.make_surface(body.sphere_shape(3.0), (2, 2)), mu,
                                         interior=True, nullspace_scale=0.5),
         interp=body.interpolate_nodal(per, q, np.array([0.3, 1.7, 2.9]), np.array([0.1, 3.0, 6.1])),
         near_W=body.near_surface_weights(per, near_t, mu, interior_jump=True),
         fnear_t=cl.X[3].mean(axis=0) + np.array([0.024, 0.018, 0.0]),
         fnear_W=fiber.near_fiber_weights(fib, cl.X[3].mean(axis=0) + np.array([0.024, 0.018, 0.0]),
                                          mu, include_doublet=True),
         fnear_eval=fiber.near_fiber_eval(fib, f, cl.X[3].mean(axis=0)
                                          + np.array([0.024, 0.018, 0.0]), mu),
         resampled=fiber.resample_to_fine(f[:, 0], np.linspace(-1, 1, 7)),
         rot_src=np.array([[0.3, -0.2, 0.1], [2.0, 1.0, -1.0]]), rot_L=np.array([[1.0, 2.0, -0.5],
                                                                                 [0.3, 0.0, 0.7]]),
         rot=kernels.rotlet_sum(tgt, np.array([[0.3, -0.2, 0.1], [2.0, 1.0, -1.0]]),
                                np.array([[1.0, 2.0, -0.5], [0.3, 0.0, 0.7]]), 0.2)[0],
         apply1=np.concatenate([kernels.stokeslet_apply(tgt[0], f[0], mu),
                                kernels.stresslet_apply(tgt[0], f[1], f[2], mu),
                                kernels.rotlet_apply(tgt[1], f[3], mu),
                                kernels.doublet_apply(tgt[2], f[4], mu)]),
         **bc_fixture(fib, Xc, Tc, mu),
         Mmat=fib.mobility_matrix(mu), Kmat=fib.kdelta_matrix(mu),
         **versions())


def tree_fixture():
    """TreeSummation (system.py:157-224) outputs: the reference tests'
    geometries plus a fiber cloud with groups, with loose and default
    parameters, and complementary_velocities through the tree backend."""
    rng = np.random.default_rng(2)
    src = rng.standard_normal((200, 3))
    src /= np.abs(src).max()
    f = rng.standard_normal((200, 3))
    far = 25.0 * np.array([[1.0, 0, 0], [0, 1.0, 0], [0.6, 0, 0.8], [-1.0, 0, 0], [0, 0, -1.0]])
    ng = lambda k: kernels.no_groups(k)   # noqa: E731
    loose = system.TreeSummation(theta=0.5, leaf_size=8, cell_tolerance=2e-2)
    out = dict(src=src, f=f, far=far,
               far_loose=loose.stokeslet(src, ng(200), f, far, ng(5), 1.0),
               far_exact=system.DirectSummation().stokeslet(src, ng(200), f, far, ng(5), 1.0))
    cl = configs.make("c1_clean", seed=0)
    X = cl.X.reshape(-1, 3)
    grp = np.repeat(np.arange(cl.X.shape[0], dtype=np.int64), cl.X.shape[1])
    fc = rng.standard_normal(X.shape)
    mid = system.TreeSummation(theta=0.6, leaf_size=16, cell_tolerance=1e-1)
    out.update(cX=X, cgrp=grp, cf=fc,
               cloud_mid=mid.stokeslet(X, grp, fc, X, grp, 1.3),
               cloud_default=system.TreeSummation().stokeslet(X, grp, fc, X, grp, 1.3),
               cloud_exact=system.DirectSummation().stokeslet(X, grp, fc, X, grp, 1.3))
    st = system.SystemState([fiber.Fiber(x, eps=1e-2, E=1.0) for x in cl.X])
    ff = rng.standard_normal(cl.X.shape)
    cv = system.complementary_velocities(st, fiber_forces=list(ff), backend=mid)
    out.update(cv_forces=ff, cv_mid=np.stack(cv.fibers))
    save("tree.npz", **out, **versions())


KIN = dict(v_grow=0.5, v_shrink=0.8, f_cat=150.0, f_res=250.0, stall_force=4.4, min_length=0.5)


def kinetics_state(pushing=True):
    """Growing aster in a small cell: dynamic instability with fast rates,
    and cortical pushing (hinged capture at the periphery) or cytoplasmic
    pulling (standoff catastrophe), per-fiber seeded RNG streams."""
    from slenderflow import system as S
    pnc = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4)))
    pts, dirs = S.aster_attachment_layout(pnc, 8, radius_factor=1.3)
    fibs = []
    for k, (x0, d) in enumerate(zip(pts, dirs)):
        fb = fiber.straight_fiber(15, x0, d, 1.0, eps=1e-2, E=1.0,
                                  growth_state=fiber.GROWING, Ldot=KIN["v_grow"],
                                  rng=np.random.default_rng(100 + k),
                                  kinetics=fiber.GrowthKinetics(**KIN))
        fb.bc_minus = fiber.ClampedToBody(0, x0, d)
        fibs.append(fb)
    per = body.Periphery(body.make_surface(body.sphere_shape(1.8), (6, 6)))
    models = ([S.CorticalPushing(stiffness=5.0, contact_distance=0.2, tau_cat=0.5)] if pushing
              else [S.CytoplasmicPulling(motor_force=0.91, motor_density=0.5)])
    return S.SystemState(fibs, [pnc], per, force_models=models)


def kinetics_fixture(name, pushing, nsteps=4, dt=1e-3):
    from slenderflow import solver as R
    st = kinetics_state(pushing)
    out = dict(dt=dt, nsteps=nsteps, init_X=np.stack([f.X for f in st.fibers]),
               init_d=np.stack([f.bc_minus.tangent for f in st.fibers]))
    params = R.GmresParams(tolerance=1e-10)
    for s_i in range(nsteps):
        R.backward_euler_step(st, dt, params)
        out[f"step{s_i}_X"] = np.stack([f.X for f in st.fibers])
        out[f"step{s_i}_T"] = np.stack([f.T for f in st.fibers])
        out[f"step{s_i}_Ldot"] = np.array([f.Ldot for f in st.fibers])
        out[f"step{s_i}_state"] = np.array([f.growth_state for f in st.fibers])
        out[f"step{s_i}_bcplus"] = np.array([f.bc_plus.kind for f in st.fibers])
        out[f"step{s_i}_tau"] = np.array([f.tau_cat for f in st.fibers])
    save(name, **out, **versions())


def layouts_fixture():
    """Attachment layouts and cloud initial condition (system.py:392-466)."""
    pnc = body.RigidParticle(body.make_surface(body.sphere_shape(0.5), (4, 4), center=(0.5, 0, 0)))
    ap, ad = system.aster_attachment_layout(pnc, 37)
    mp, md = system.mtoc_attachment_layout(pnc, 36)
    cl = system.cloud_init(20, 3.0, 1.0, 1e-2, 1.0, seed=4)
    save("layouts.npz", aster_p=ap, aster_d=ad, mtoc_p=mp, mtoc_d=md,
         cloud_X=np.stack([f.X for f in cl.fibers]), **versions())


def spectral_fixture():
    """Spectral API values (spectral.py:24-154) on a p = 31 grid."""
    from slenderflow import spectral as R
    g = R.ChebyshevGrid(31)
    X = configs.make("c1_clean", seed=0).X[5]
    v = np.sin(3 * g.nodes) + 0.2 * g.nodes ** 5
    s, sa, L = R.arclength_map(X, g)
    save("spectral.npz", nodes=g.nodes, weights=g.weights, D=g.D, X=X, s=s, s_alpha=sa, L=L, v=v,
         dv=R.cheb_diff(v, g), iv=R.cheb_integrate(v, g), cv=R.cheb_transform(v),
         interp=np.array([R.cheb_interp(v, a) for a in (-1.0, -0.37, 0.3, 1.0)]), **versions())


def shapes_fixture():
    """Non-spherical profile meshes (body.py:37-72) and a near-surface map on
    one of them (exercises the golden-section nearest point on R(theta))."""
    out = {}
    for k in ("s1", "s2", "s3"):
        m = body.make_surface(body.named_shape(k, 2.0), (6, 8), center=(0.1, -0.2, 0.3))
        out.update({f"{k}_nodes": m.nodes, f"{k}_normals": m.normals, f"{k}_weights": m.weights})
    per = body.make_surface(body.s1_shape(2.0), (6, 8))
    t = np.array([[0.2, 0.1, 1.2], [1.5, 0.3, -0.1]])
    rho = [np.linalg.norm(x) for x in t]
    out["near_t"] = t
    out["near_W"] = np.stack([body.near_surface_weights(per, x, 1.0, interior_jump=True)
                              - body.plain_surface_weights(per, x, 1.0) for x in t])
    out["near_ns"] = np.array([[*body.nearest_surface_point(per, x)[:2],
                                body.nearest_surface_point(per, x)[3]] for x in t])
    print("  shapes: target radii", rho)
    save("shapes.npz", **out, **versions())


if __name__ == "__main__":
    which = sys.argv[1:] or ["pairs", "operator", "surfaces", "steps"]
    if "pairs" in which:
        pairs_small()
    if "operator" in which:
        operator_fixture("c1_near.npz", configs.make("c1", seed=0))
        operator_fixture("c1_clean.npz", configs.make("c1_clean", seed=0))
    if "surfaces" in which:
        surfaces_fixture()
        near_surface_fixture()


    if "steps" in which:
        steps_all()
    if "api" in which:
        api_ops_fixture()
    if "tree" in which:
        tree_fixture()
    if "mixed" in which:
        steps_mixed()
    if "shapes" in which:
        shapes_fixture()
        layouts_fixture()
        spectral_fixture()
    if "kinetics" in which:
        kinetics_fixture("step_pushing.npz", True)
        kinetics_fixture("step_pulling.npz", False)
