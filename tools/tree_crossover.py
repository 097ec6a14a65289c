"""Tree (octree monopole + dipole, the reference's TreeSummation backend on
the device) vs all-pairs for the fiber Stokeslet sum of sedimenting clouds
of growing size at C3's density: time per evaluation
(CUDA events, after a warm-up that also builds the host topology) and the
relative L2 difference from the exact all-pairs sum, for the reference's
default gates and for looser ones.
Usage: python tools/tree_crossover.py [n_fibers ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, kernels, system  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [512, 2048, 4096, 16384]
dev = torch.device("cuda")


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


for nfib in sizes:
    R = 10.0 * (nfib / 4096.0) ** (1.0 / 3.0)          # C3 density
    cl = configs.make("c3", seed=0, n_fibers=nfib, size=R)
    X = torch.as_tensor(cl.X.reshape(-1, 3), device=dev).contiguous()
    N = X.shape[0]
    grp = torch.arange(nfib, device=dev).repeat_interleave(cl.n_nodes).contiguous()
    f = torch.as_tensor(np.random.default_rng(1).standard_normal((N, 3)), device=dev).contiguous()
    pref = 1.0 / (8.0 * np.pi)
    t_dir, (u_dir, _) = timed(lambda: kernels.stokeslet_sum(X, grp, X, grp, f, pref))
    rec = {"n_fibers": nfib, "points": N, "direct_ms": t_dir,
           "direct_pairs_per_s": (N * N - nfib * cl.n_nodes ** 2) / (t_dir * 1e-3)}
    for name, kw in (("reference_gates", {}), ("theta0.5_tol1e-4", dict(cell_tolerance=1e-4)),
                     ("theta0.7_tol1e-3", dict(theta=0.7, cell_tolerance=1e-3)),
                     ("theta0.5_tol1e-1", dict(theta=0.5, cell_tolerance=1e-1)),
                     ("theta0.5_tol1", dict(theta=0.5, cell_tolerance=1.0))):
        tb = system.TreeSummation(**kw)
        t_tree, u_tree = timed(lambda: tb.stokeslet(X, grp, f, X, grp, 1.0))
        rec[name] = {"ms": t_tree, "speedup": t_dir / t_tree,
                     "rel_l2_vs_direct": float((u_tree - u_dir).norm() / u_dir.norm())}
    print(json.dumps(rec), flush=True)
