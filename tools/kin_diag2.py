import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import golden
from test_gpu_kinetics import build
from paper_1602_05650_b200 import solver
from oracle.ops import rel_l2
r = np.load("tools/_diag/ref_kin_step1.npz")
g = golden("step_pushing.npz")
st = build(g, True)
params = solver.GmresParams(tolerance=1e-10)
st = solver.backward_euler_step(st, 0.05, params)
X = np.stack([f.X for f in st.fibers])
print("X after step0", rel_l2(X, r["X"]), "Ldot", np.abs(np.array([f.Ldot for f in st.fibers]) - r["Ldot"]).max())
print("att", np.abs(np.stack([getattr(f.bc_plus, "attachment", np.zeros(3)) for f in st.fibers]) - r["att"]).max())
print("q", rel_l2(st.particles[0].q, r["q"]), "q0", rel_l2(st.periphery.q, r["q0"]), "U", np.abs(st.particles[0].U - r["U"]).max())
op, rhs = solver.assemble_step_operator(st, 0.05)
print("Au", rel_l2(op.apply(r["u"]), r["Au"]), "rhs", rel_l2(rhs.cpu().numpy(), r["rhs"]), "block0", rel_l2(op.fiber_blocks[0].cpu().numpy(), r["block0"]))
prec = solver.Preconditioner(op)
print("Mv", rel_l2(prec.apply(r["u"]), r["Mv"]))
x, it, hist = solver.gmres_solve(op, prec, rhs, params)
print("x", rel_l2(x.cpu().numpy(), r["x"]), it, r["it"])
# per-block error
lay = op.layout
xx = x.cpu().numpy()
for m in range(8):
    sl = lay.fiber_block[m]; print(m, rel_l2(xx[sl], r["x"][sl]))
print("surf", rel_l2(xx[:lay.fib_off], r["x"][:lay.fib_off]))
