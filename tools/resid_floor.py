"""True residual of a 1e-10 GMRES solve on a 64-fiber p=63 cloud (the operator's
rounding floor); optional argument: another libsf_b200.so to compare."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1602_05650_b200 import _native
if len(sys.argv) > 1:
    _native.LIB = sys.argv[1]
import numpy as np
from paper_1602_05650_b200 import configs, solver
st = configs.cloud_state("c3_scaled", n_fibers=64)
op, rhs = solver.assemble_step_operator(st, 5e-3)
prec = solver.Preconditioner(op)
x, it, hist = solver.gmres_solve(op, prec, rhs, solver.GmresParams(tolerance=1e-10))
res = op.apply(x.cpu().numpy()) - rhs.cpu().numpy()
print(sys.argv[1:] or "new", it, hist[-1], np.linalg.norm(res) / np.linalg.norm(rhs.cpu().numpy()))
# operator rounding floor: A(x) vs the same x split in two halves
xa = x.cpu().numpy(); h = 0.5 * xa
fl = op.apply(h) + op.apply(xa - h) - op.apply(xa)
print("  linearity floor |A(x/2)+A(x-x/2)-A(x)|/|rhs|", np.linalg.norm(fl) / np.linalg.norm(rhs.cpu().numpy()))
