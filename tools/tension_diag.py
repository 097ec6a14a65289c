"""Per-block parity of the step operator at the BASELINE orders (GPU):
A u, rhs and M v against the reference's golden vectors, split into the
fiber velocity rows (X), the inextensibility rows (T) and the surface rows,
so a block whose rows are small next to the 1/dt-scaled velocity rows is not
hidden inside a whole-vector relative L2."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from test_gpu_baseline_steps import state_from  # noqa: E402
from conftest import golden  # noqa: E402
from paper_1602_05650_b200 import solver  # noqa: E402


def rl(a, b):
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / d if d else np.linalg.norm(a)


def blocks(lay):
    xi = np.concatenate([np.arange(s.start, s.stop) for s in lay.X])
    ti = np.concatenate([np.arange(s.start, s.stop) for s in lay.T])
    si = np.arange(0, lay.fib_off)
    n = lay.X[0].stop - lay.X[0].start
    n = n // 3
    # per fiber rows: X rows 0..3n, T rows 3n..4n; BC rows replace vel rows 0,1,n-1,n-2 and inext 0,n-1
    bc = []
    for sx, stt in zip(lay.X, lay.T):
        for r in (0, 1, n - 2, n - 1):
            bc.extend(range(sx.start + 3 * r, sx.start + 3 * r + 3))
        bc.extend([stt.start, stt.start + n - 1])
    bc = np.array(bc)
    xin = np.setdiff1d(xi, bc)
    tin = np.setdiff1d(ti, bc)
    return dict(X_interior=xin, T_interior=tin, BC=bc, surface=si)


def main(name):
    g = golden(name)
    st = state_from(g)
    op, rhs = solver.assemble_step_operator(st, float(g["dt"]))
    n = op.layout.size
    u = np.random.default_rng(int(g["seed_u"])).standard_normal(n)
    v = np.random.default_rng(int(g["seed_v"])).standard_normal(n)
    Au = op.apply(u)
    r = rhs.cpu().numpy()
    Mv = solver.Preconditioner(op).apply(v)
    for k, idx in blocks(op.layout).items():
        if idx.size == 0:
            continue
        print(f"{name:22s} {k:11s} rows {idx.size:7d}  Au {rl(Au[idx], g['apply_Au'][idx]):.2e}"
              f"  rhs {rl(r[idx], g['rhs'][idx]):.2e}  Mv {rl(Mv[idx], g['prec_Mv'][idx]):.2e}"
              f"  |Au| {np.linalg.norm(g['apply_Au'][idx]):.2e}", flush=True)
    params = solver.GmresParams(tolerance=float(g["tol"]))
    st, info = solver.backward_euler_step(st, float(g["dt"]), params, return_info=True)
    X = np.stack([f.X for f in st.fibers])
    T = np.stack([f.T for f in st.fibers])
    print(f"{name}: step0 iters {info['iterations']} vs {int(g['iters_0'])}; X {rl(X, g['step0_X']):.2e}"
          f" T {rl(T, g['step0_T']):.2e}", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["bstep_c1.npz"]:
        main(nm)
