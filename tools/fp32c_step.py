"""Implicit step with the FP32-compute / FP64-accumulate fiber pair sums:
convergence and difference from the FP64 step (usage: config tol)."""
import copy
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3_scaled"
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
st0 = configs.cloud_state(cfg)
res = {}
for prec in ("fp64", "fp32c"):
    st = copy.deepcopy(st0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        st, info = solver.backward_euler_step(st, 5e-3, solver.GmresParams(tolerance=tol, max_iterations=200),
                                              return_info=True, precision=prec)
        torch.cuda.synchronize()
        res[prec] = np.stack([f.X for f in st.fibers])
        disp = res[prec] - np.stack([f.X for f in st0.fibers])
        res[prec + "_d"] = disp
        print(prec, f"{time.perf_counter() - t0:.2f} s", info["iterations"], f"{info['history'][-1]:.2e}",
              flush=True)
    except solver.NonconvergenceError as e:
        print(prec, "nonconvergence", e.iterations, e.residuals[-5:], flush=True)
if "fp32c" in res:
    d = res["fp32c_d"] - res["fp64_d"]
    print("displacement rel diff", np.linalg.norm(d) / np.linalg.norm(res["fp64_d"]))
