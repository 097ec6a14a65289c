"""Target-block sharding of the HI operator across GPUs (one process per GPU).

SURVEY.md §8(e): every target's output is independent, so rank r owns a
contiguous block of fibers (its nodes are its targets and its unknowns).
Once per matvec each rank contributes its fibers' force densities and an
all-gather (NCCL over NVLink/NVSwitch) gives every rank the full source
strengths; each rank then evaluates its target block against all sources in
the same fixed order as on one GPU, so per-target sums are bitwise identical
at any world size.  The distributed implicit step built on it (sharded block
rows, gathered or all-reduced GMRES) is dsolver.py.
"""

import os

import numpy as np
import torch
import torch.distributed as dist

# modelled cost of a symmetric-kernel cell on the checked path and of a
# diagonal-task cell, relative to a check-free both-ways cell (measured with
# SF_SYM_NOFAST, tools/sym_split_balance.py)
SYM_CHECKED_COST = float(os.environ.get("SF_SYM_CHECKED_COST", "1.11"))
SYM_DIAG_COST = float(os.environ.get("SF_SYM_DIAG_COST", "0.75"))


def sym_task_costs(X, groups, N, n, mode):
    """Per-task modelled cost (host array) of the symmetric fiber x fiber
    evaluation of the positions X (device (N,3)): sf_sym_task_costs replays
    the task kernel's check-free / checked slab-pair decisions."""
    import ctypes

    from . import _native
    lib = _native.load(require_device=True)
    nt = int(lib.sf_sym_task_count(N, n, mode))
    cost = torch.empty(nt, dtype=torch.float64, device=X.device)
    _native.call("sf_sym_task_costs", X.data_ptr(), groups.data_ptr() if groups is not None else None,
                 N, n, mode, SYM_CHECKED_COST, SYM_DIAG_COST, cost.data_ptr(),
                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    return cost.cpu().numpy()


def cost_split(costs, world):
    """[(t0, count)] per rank: contiguous task ranges of equal modelled cost
    (boundaries where the cumulative cost crosses r/world of the total).
    A pure function of the costs, so every rank computes the same split."""
    c = np.cumsum(np.asarray(costs, dtype=float))
    total = c[-1] if c.size else 0.0
    bounds = [0] + [int(np.searchsorted(c, total * r / world, side="left")) + 1
                    for r in range(1, world)] + [c.size]
    bounds = np.maximum.accumulate(np.minimum(bounds, c.size))
    return [(int(bounds[r]), int(bounds[r + 1] - bounds[r])) for r in range(world)]


def pair_costs(N, n, mode):
    """Per-task pair-geometry count (2 n_g n_h both ways, n_g^2 on the
    diagonal), tasks row-major {g <= h}: the library's pair-count model."""
    from . import _native
    M = int(_native.load().sf_sym_unit_size(N, n, mode))
    G = -(-N // M)
    nu = np.minimum(M, N - M * np.arange(G)).astype(float)
    rows = [np.concatenate([[nu[g] * nu[g]], 2.0 * nu[g] * nu[g + 1:]]) for g in range(G)]
    return np.concatenate(rows)


def pair_split(N, n, mode, world):
    """[(t0, count)] per rank balanced by pair count (SF_SYM_SPLIT=pairs)."""
    return cost_split(pair_costs(N, n, mode), world)


def task_ranges(X, groups, N, n, mode, world):
    """The rank task split used by the multi-GPU symmetric evaluation:
    by modelled cost (default) or by pair count (SF_SYM_SPLIT=pairs)."""
    if os.environ.get("SF_SYM_SPLIT", "cost") == "pairs":
        return pair_split(N, n, mode, world)
    return cost_split(sym_task_costs(X, groups, N, n, mode), world)


def shard_range(nf, rank, world):
    """Fibers [f0, f0 + count) owned by `rank` (ceil-sized contiguous blocks)."""
    per = -(-nf // world)
    f0 = min(nf, rank * per)
    return f0, min(nf, f0 + per) - f0


class ShardedHIOperator:
    """Wraps a shard-local operator (FiberHIOperator(shard=(rank, world)) or
    any object with nf, n, f0, nown and apply(f_full) -> (u_nl, u_self))."""

    def __init__(self, local_op, group=None):
        self.op = local_op
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.per = -(-local_op.nf // self.world)
        dev = getattr(local_op, "device", torch.device("cpu"))
        n = local_op.n
        self._f_full = torch.zeros((self.world * self.per, n, 3), dtype=torch.float64, device=dev)
        self._f_pad = torch.zeros((self.per, n, 3), dtype=torch.float64, device=dev)

    def gather_sources(self, f_local):
        """All-gather every rank's (nown, n, 3) force densities -> (nf, n, 3)."""
        nf = self.op.nf
        if self.world == 1:
            return f_local.reshape(nf, self.op.n, 3)
        self._f_pad.zero_()
        self._f_pad[: f_local.shape[0]].copy_(f_local)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(self._f_full, self._f_pad, group=self.group)
        else:
            parts = list(self._f_full.chunk(self.world))
            dist.all_gather(parts, self._f_pad, group=self.group)
        return self._f_full[:nf]

    def apply(self, f_local, out_nl=None, out_self=None, self_terms=True):
        """One matvec of the HI operator on this rank's target block.

        Symmetric path (FP64, >= 8192 points): every rank evaluates its share
        of the unit-pair tasks for all points, a reduce-scatter sums the
        partials onto the target blocks, then near maps and self terms run
        locally.  Otherwise each rank evaluates its targets against all
        sources (direct path)."""
        f_full = self.gather_sources(f_local)
        op = self.op
        if getattr(op, "symmetric_shard", False):
            part = op.symmetric_partial(f_full)
            u_own = self.reduce_scatter_points(part, out_nl)
            return op.finish_own(u_own, f_full, out_self=out_self, self_terms=self_terms)
        return op.apply(f_full, out_nl=out_nl, out_self=out_self, self_terms=self_terms)

    def reduce_scatter_points(self, part, out=None):
        """Sum (N,3) per-rank partials over ranks; return this rank's (Nown,3)."""
        n = self.op.n
        rows = self.per * n
        full = torch.zeros((self.world * rows, 3), dtype=part.dtype, device=part.device)
        full[: part.shape[0]].copy_(part)
        mine = torch.empty((rows, 3), dtype=part.dtype, device=part.device)
        if dist.get_backend(self.group) == "nccl":
            dist.reduce_scatter_tensor(mine, full, group=self.group)
        else:
            dist.all_reduce(full, group=self.group)
            mine.copy_(full[self.rank * rows:(self.rank + 1) * rows])
        nown = self.op.Nown
        if out is None:
            return mine[:nown].contiguous()
        out.copy_(mine[:nown])
        return out

    def gather_targets(self, u_local):
        """All-gather per-rank (Nown,3) outputs into the global (N,3) array."""
        if self.world == 1:
            return u_local
        n = self.op.n
        pad = torch.zeros((self.per * n, 3), dtype=u_local.dtype, device=u_local.device)
        pad[: u_local.shape[0]].copy_(u_local)
        full = torch.zeros((self.world * self.per * n, 3), dtype=u_local.dtype,
                           device=u_local.device)
        if dist.get_backend(self.group) == "nccl":
            dist.all_gather_into_tensor(full, pad, group=self.group)
        else:
            dist.all_gather(list(full.chunk(self.world)), pad, group=self.group)
        return full[: self.op.nf * n]
