"""Distributed implicit step (dsolver.py) with 2-3 ranks emulated as threads
on one GPU (ThreadComm: host-side exchanges only, no kernel waits on another
rank).  Each rank's rows must equal the single-GPU operator's rows, and the
sharded step must reproduce the reference's golden steps (tolerances of
test_gpu_solver.py)."""

import copy
import threading

import numpy as np
import pytest

from conftest import golden
from oracle.ops import rel_l2
from paper_1602_05650_b200 import dsolver, solver
from test_gpu_solver import CASES

pytestmark = pytest.mark.gpu


def run_ranks(world, fn):
    """fn(comm) on `world` threads, each with its own CUDA stream."""
    import torch
    hub = dsolver.ThreadHub(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = fn(dsolver.ThreadComm(hub, r))
                torch.cuda.current_stream().synchronize()
        except BaseException as e:       # noqa: BLE001 - re-raised below
            errs.append(e)
            hub.barrier.abort()
    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("symmetric", [False, True])
@pytest.mark.parametrize("name", sorted(CASES))
def test_dist_rows_match_single_gpu(cuda, name, world, symmetric):
    import torch
    g = golden(name)
    st = CASES[name](g)
    dt = float(g["dt"])
    op1 = solver.BlockOperator(st, dt)
    rng = np.random.default_rng(7)
    u = rng.standard_normal(op1.layout.size)
    ref = op1.apply(u)
    ref_rhs = op1.rhs()

    def fn(comm):
        op = dsolver.DistBlockOperator(copy.deepcopy(st), dt, comm, symmetric=symmetric)
        a = op.rows_device(torch.as_tensor(u, device=cuda), False).cpu().numpy()
        b = op.rhs_device().cpu().numpy()
        return op.owned, a, b
    for owned, a, b in run_ranks(world, fn):
        for lo, hi in owned:
            assert rel_l2(a[lo:hi], ref[lo:hi]) < 1e-12
            assert rel_l2(b[lo:hi], ref_rhs[lo:hi]) < 1e-12


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_dist_steps_match_reference(cuda, name, world):
    g = golden(name)
    st0 = CASES[name](g)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    dt = float(g["dt"])

    def fn(comm):
        st = copy.deepcopy(st0)
        res = []
        for _ in range(int(g["nsteps"])):
            st, info = dsolver.dist_backward_euler_step(st, dt, comm, params, return_info=True)
            res.append((np.stack([f.X for f in st.fibers]), np.stack([f.T for f in st.fibers]),
                        info["iterations"]))
        return res
    results = run_ranks(world, fn)
    for s in range(int(g["nsteps"])):
        X, T, it = results[0][s]
        for r in range(1, world):                      # replicated state agrees
            assert np.array_equal(results[r][s][0], X)
        ref = g[f"step{s}_X"]
        assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-8
        assert rel_l2(T, g[f"step{s}_T"]) < 1e-6
        assert abs(it - int(g[f"iters_{s}"])) <= 1


def test_dist_kinetics_steps_match_reference(cuda):
    """Kinetics + cortical pushing over 2 emulated ranks: replicated host
    state, same RNG streams, same transitions as the reference."""
    from test_gpu_kinetics import build
    g = golden("step_pushing.npz")
    params = solver.GmresParams(tolerance=1e-10)

    def fn(comm):
        st = build(g, True)
        res = []
        for _ in range(int(g["nsteps"])):
            st = dsolver.dist_backward_euler_step(st, float(g["dt"]), comm, params)
            res.append((np.stack([f.X for f in st.fibers]), [f.growth_state for f in st.fibers],
                        [f.bc_plus.kind for f in st.fibers]))
        return res
    out = run_ranks(2, fn)
    for s in range(int(g["nsteps"])):
        X, states, bcs = out[0][s]
        assert np.array_equal(out[1][s][0], X)
        assert states == list(g[f"step{s}_state"]) and bcs == list(g[f"step{s}_bcplus"])
        ref = g[f"step{s}_X"]
        assert np.linalg.norm(X - ref) / np.linalg.norm(ref) < 1e-8


def test_dist_rows_mid_size_confined(cuda):
    """A confined aster large enough for the symmetric, cross and symmetric
    double-layer kernels on one GPU (16,384 fiber points, 9,216-node
    periphery): rows of 2 emulated ranks equal the single-GPU rows."""
    import torch
    from paper_1602_05650_b200 import configs
    st = configs.confined_aster(n_fibers=512, periphery_res=(24, 24), periphery_radius=2.5)
    op1 = solver.BlockOperator(st, 1e-3)
    u = np.random.default_rng(2).standard_normal(op1.layout.size)
    ref = op1.apply(u)

    def fn(comm):
        op = dsolver.DistBlockOperator(copy.deepcopy(st), 1e-3, comm)
        return op.owned, op.rows_device(torch.as_tensor(u, device=cuda), False).cpu().numpy()
    for owned, a in run_ranks(2, fn):
        for lo, hi in owned:
            assert rel_l2(a[lo:hi], ref[lo:hi]) < 1e-12


def test_torch_comm_nccl_single_rank_step(cuda):
    """The NCCL code path of TorchComm (all_gather_into_tensor,
    reduce_scatter_tensor, broadcast, all_reduce) in a world-size-1 process
    group on the box: the distributed step reproduces the golden step."""
    import socket

    import torch.distributed as dist
    g = golden("step_confined.npz")
    st = CASES["step_confined.npz"](g)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=cuda)
    try:
        comm = dsolver.TorchComm()
        assert comm.nccl
        params = solver.GmresParams(tolerance=float(g["tol"]))
        st, info = dsolver.dist_backward_euler_step(st, float(g["dt"]), comm, params,
                                                    return_info=True, symmetric=True)
    finally:
        dist.destroy_process_group()
    X = np.stack([f.X for f in st.fibers])
    assert np.linalg.norm(X - g["step0_X"]) / np.linalg.norm(g["step0_X"]) < 1e-8
    assert abs(info["iterations"] - int(g["iters_0"])) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_dist_body_coupled_preconditioner_matches_single_gpu(cuda, world):
    """DistPreconditioner(body_coupling=True) on the golden aster: every rank's
    owned entries of M v equal the single-GPU body-coupled preconditioner's
    (the particle block is replicated, the fiber blocks sharded)."""
    import torch
    g = golden("step_aster.npz")
    st = CASES["step_aster.npz"](g)
    dt = float(g["dt"])
    op1 = solver.BlockOperator(st, dt)
    rng = np.random.default_rng(11)
    v = rng.standard_normal(op1.layout.size)
    ref = solver.Preconditioner(op1, body_coupling=True).apply(v)

    def fn(comm):
        op = dsolver.DistBlockOperator(copy.deepcopy(st), dt, comm)
        prec = dsolver.DistPreconditioner(op, body_coupling=True)
        vd = torch.as_tensor(v, device="cuda")
        rows = vd.clone()
        if comm.rank:                      # particle rows of v live on rank 0 only
            rows[:op.layout.fib_off] = 0.0
        out = prec.apply_device(rows)
        return [(a, b, out[a:b].cpu().numpy()) for a, b in op.owned]

    for per_rank in run_ranks(world, fn):
        for a, b, got in per_rank:
            assert rel_l2(got, ref[a:b]) < 1e-11, (a, b)


def test_dist_body_coupled_step_matches_golden(cuda):
    """The distributed step with the body-coupled preconditioner (2 ranks)
    reproduces the reference's golden aster step; its iteration count equals
    the single-GPU body-coupled solve's (+-1)."""
    g = golden("step_aster.npz")
    st0 = CASES["step_aster.npz"](g)
    dt = float(g["dt"])
    params = solver.GmresParams(tolerance=float(g["tol"]))
    _, info1 = solver.backward_euler_step(copy.deepcopy(st0), dt, params, return_info=True,
                                          body_coupling=True)

    def fn(comm):
        st, info = dsolver.dist_backward_euler_step(copy.deepcopy(st0), dt, comm, params,
                                                    return_info=True, body_coupling=True)
        return np.stack([f.X for f in st.fibers]), info["iterations"]

    for X, iters in run_ranks(2, fn):
        assert np.linalg.norm(X - g["step0_X"]) / np.linalg.norm(g["step0_X"]) < 1e-8
        assert abs(iters - info1["iterations"]) <= 1
