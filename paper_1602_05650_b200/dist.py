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

import torch
import torch.distributed as dist


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
