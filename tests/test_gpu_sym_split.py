"""Multi-GPU split of the symmetric fiber-pair evaluation,
checked with the ranks emulated on one GPU: the unit-pair tasks are split
into contiguous ranges of equal MODELLED cost (sf_sym_task_costs replays
the task kernel's check-free / checked slab-pair decisions), every split
covers each task exactly once, and the ranks' partials sum to the one-GPU
result."""

import numpy as np
import pytest
import torch

from paper_1602_05650_b200 import _native, configs, dist
from paper_1602_05650_b200.operator import FiberHIOperator

pytestmark = pytest.mark.gpu


def _op(cfg, world, cuda):
    if cfg == "c2":
        st = configs.aster(n_fibers=1024)
        X, eps = np.stack([f.X for f in st.fibers]), 1e-2
    else:
        cl = configs.make(cfg, seed=0)
        X, eps = cl.X, cl.eps
    return FiberHIOperator(X, eps, device=cuda, shard=(0, world)), X


def test_c5_cost_split_is_balanced_over_8_ranks(cuda):
    op, _ = _op("c5", 8, cuda)
    costs = dist.sym_task_costs(op.X.reshape(-1, 3), op.groups, op.N, op.n, op.mode)
    T = int(_native.load().sf_sym_task_count(op.N, op.n, op.mode))
    assert costs.size == T and np.all(costs > 0)
    split = dist.cost_split(costs, 8)
    assert split[0][0] == 0 and sum(c for _, c in split) == T
    assert all(a + c == b for (a, c), (b, _) in zip(split, split[1:]))
    model = np.array([costs[t0:t0 + c].sum() for t0, c in split])
    assert model.max() / model.mean() - 1.0 < 0.02
    # pairs of the shares add up to every non-excluded ordered pair
    lib = _native.load()
    pairs = sum(int(lib.sf_sym_range_pairs(op.N, op.n, op.mode, t0, c)) for t0, c in split)
    assert pairs == op.N * op.N - op.nf * op.n * op.n


@pytest.mark.parametrize("cfg,world", [("c2", 3), ("c3_scaled", 8)])
def test_cost_split_partials_sum_to_the_one_gpu_result(cuda, cfg, world):
    op, X = _op(cfg, world, cuda)
    f = torch.as_tensor(np.random.default_rng(2).standard_normal(X.shape), device=cuda)
    f = f.reshape(-1, 3).contiguous()
    total = sum(op.symmetric_partial(f, rank=r, world=world) for r in range(world))
    one = FiberHIOperator(X, op.eps.cpu().numpy(), device=cuda, shard=(0, 1))
    full = one.symmetric_partial(f, world=1)
    assert float((total - full).norm() / full.norm()) < 1e-14


def test_cost_model_beats_pair_count_on_an_aster(cuda):
    """Near the centrosome whole slab pairs take the checked path; the cost
    split accounts for it, the pair-count split does not."""
    op, _ = _op("c2", 8, cuda)
    costs = dist.sym_task_costs(op.X.reshape(-1, 3), op.groups, op.N, op.n, op.mode)
    imb = {}
    for name, split in (("pairs", dist.pair_split(op.N, op.n, op.mode, 8)),
                        ("cost", dist.cost_split(costs, 8))):
        m = np.array([costs[t0:t0 + c].sum() for t0, c in split])
        imb[name] = m.max() / m.mean() - 1.0
    assert imb["cost"] <= imb["pairs"] + 1e-12
    assert imb["cost"] < 0.02
