import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import golden
from test_gpu_kinetics import build
from paper_1602_05650_b200 import solver
g = golden("step_pushing.npz")
st = build(g, True)
params = solver.GmresParams(tolerance=1e-10)
for s in range(4):
    st = solver.backward_euler_step(st, float(g["dt"]), params)
    X = np.stack([f.X for f in st.fibers]); ref = g[f"step{s}_X"]
    print(s, "Xrel", np.linalg.norm(X-ref)/np.linalg.norm(ref), "tipdiff", np.abs(X[:,0]-ref[:,0]).max(axis=1),
          "Ldot", np.abs(np.array([f.Ldot for f in st.fibers]) - g[f"step{s}_Ldot"]).max(),
          [f.growth_state for f in st.fibers] == list(g[f"step{s}_state"]))
