"""Multi-rank host logic of the target-block sharded HI operator, world size 2
on the CPU with gloo.  Each rank evaluates its target block with the CPU
oracle standing in for the device kernel (the only thing that differs on the
B200 is that local evaluator); the gathered result must equal the
single-process evaluation exactly, row for row."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ops, pairs
from paper_1602_05650_b200 import configs
from paper_1602_05650_b200.dist import ShardedHIOperator, shard_range


class OracleShardOperator:
    """Shard-local operator with the FiberHIOperator interface, on the CPU."""

    def __init__(self, X, eps, rank, world):
        self.X = X
        self.nf, self.n = X.shape[0], X.shape[1]
        self.f0, self.nown = shard_range(self.nf, rank, world)
        self.device = torch.device("cpu")
        self.eps = eps
        geos = [ops.geometry(X[m]) for m in range(self.nf)]
        self.w = np.concatenate([g["weights"] for g in geos])
        self.c = np.repeat([(eps * g["L"]) ** 2 / 2.0 for g in geos], self.n)

    def apply(self, f_full, out_nl=None, out_self=None, self_terms=True):
        f = f_full.numpy().reshape(-1, 3)
        src = self.X.reshape(-1, 3)
        grp = np.repeat(np.arange(self.nf, dtype=np.int64), self.n)
        lo, hi = self.f0 * self.n, (self.f0 + self.nown) * self.n
        s = self.w[:, None] * f
        pref = 1.0 / (8.0 * np.pi)
        u1, _ = pairs.stokeslet_sum(src[lo:hi], grp[lo:hi], src, grp, s, pref)
        u2, _ = pairs.doublet_sum(src[lo:hi], grp[lo:hi], src, grp, self.c[:, None] * s, pref)
        return torch.as_tensor(u1 + u2), None


class SymmetricShardOperator(OracleShardOperator):
    """Stand-in for the symmetric multi-GPU form: each rank returns a partial
    for EVERY point (here: the full oracle sum split by a fixed per-rank
    weight) and the dist layer must reduce-scatter them."""

    symmetric_shard = True

    def __init__(self, X, eps, rank, world):
        super().__init__(X, eps, rank, world)
        self.rank, self.world = rank, world
        self.Nown = self.nown * self.n

    def symmetric_partial(self, f_full):
        full = OracleShardOperator(self.X, self.eps, 0, 1).apply(f_full)[0]
        return full * (0.25 if self.rank == 0 else 0.75 / (self.world - 1))

    def finish_own(self, u_own, f_full, out_self=None, self_terms=True):
        return u_own, None


def _sym_worker(rank, world, port, X, eps, F, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op = SymmetricShardOperator(X, eps, rank, world)
        sop = ShardedHIOperator(op)
        u_own, _ = sop.apply(torch.as_tensor(F[op.f0:op.f0 + op.nown]))
        full = sop.gather_targets(u_own)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_symmetric_reduce_scatter():
    cloud = configs.fiber_cloud(9, 15, eps=1e-2, region="cube", size=1.5, seed=5,
                                clear=configs.clean_clear(15), check="node")
    F = configs.forces(cloud, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, 2, port, cloud.X, cloud.eps, F, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, _ = ops.fiber_operator(cloud.X, F, cloud.eps)
    assert ops.rel_l2(got, ref) < 1e-14


def _worker(rank, world, port, X, eps, F, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        op = OracleShardOperator(X, eps, rank, world)
        sop = ShardedHIOperator(op)
        f_local = torch.as_tensor(F[op.f0:op.f0 + op.nown])
        u_local, _ = sop.apply(f_local)
        full = sop.gather_targets(u_local)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nf", [10, 9])   # even and uneven shards
def test_two_rank_sharded_operator_matches_single_process(nf):
    cloud = configs.fiber_cloud(nf, 15, eps=1e-2, region="cube", size=1.5, seed=4,
                                clear=configs.clean_clear(15), check="node")
    F = configs.forces(cloud, seed=2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cloud.X, cloud.eps, F, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, _ = ops.fiber_operator(cloud.X, F, cloud.eps)
    one = OracleShardOperator(cloud.X, cloud.eps, 0, 1).apply(torch.as_tensor(F))[0].numpy()
    assert np.array_equal(got, one)          # sharding changes no row bitwise
    assert ops.rel_l2(got, ref) < 1e-14


def test_shard_ranges_cover_all_fibers():
    for nf in (1, 7, 64, 16384):
        for world in (1, 2, 3, 8):
            spans = [shard_range(nf, r, world) for r in range(world)]
            covered = [m for f0, c in spans for m in range(f0, f0 + c)]
            assert covered == list(range(nf))


# ----------------------------------------------- dsolver Comm semantics ----
def _comm_ops(comm):
    """The four collectives dsolver uses, on rank-dependent inputs."""
    from paper_1602_05650_b200.dsolver import ThreadComm  # noqa: F401 (import check)
    r, w = comm.rank, comm.world
    a = torch.arange(6, dtype=torch.float64) * (r + 1)
    comm.all_reduce_sum(a)
    b = torch.full((3,), float(r + 10), dtype=torch.float64)
    comm.broadcast(b, src=0)
    c = torch.empty((2 * w, 3), dtype=torch.float64)
    comm.all_gather(c, torch.full((2, 3), float(r), dtype=torch.float64))
    d = torch.empty((2, 3), dtype=torch.float64)
    comm.reduce_scatter_sum(d, torch.arange(6 * w, dtype=torch.float64).reshape(2 * w, 3) + r)
    return [x.numpy().copy() for x in (a, b, c, d)]


def _expected(r, w):
    a = np.arange(6.0) * sum(k + 1 for k in range(w))
    b = np.full(3, 10.0)
    c = np.repeat(np.arange(w, dtype=float), 2)[:, None] * np.ones(3)
    d = sum(np.arange(6.0 * w).reshape(2 * w, 3) + k for k in range(w))[2 * r:2 * r + 2]
    return [a, b, c, d]


def _comm_worker(rank, world, port, q):
    from paper_1602_05650_b200.dsolver import TorchComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _comm_ops(TorchComm())))
    finally:
        dist.destroy_process_group()


def test_torch_comm_collectives_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        for x, e in zip(got[r], _expected(r, 2)):
            assert np.array_equal(x, e)


@pytest.mark.parametrize("world", [2, 3])
def test_thread_comm_collectives(world):
    import threading
    from paper_1602_05650_b200.dsolver import ThreadComm, ThreadHub
    hub = ThreadHub(world)
    got = [None] * world
    th = [threading.Thread(target=lambda r=r: got.__setitem__(r, _comm_ops(ThreadComm(hub, r))))
          for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    for r in range(world):
        for x, e in zip(got[r], _expected(r, world)):
            assert np.array_equal(x, e)
