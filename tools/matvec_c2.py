import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_1602_05650_b200 import configs, solver
from paper_1602_05650_b200.system import InteractionCache
st = configs.aster(n_fibers=1024)
cache = InteractionCache(st)
op, rhs = solver.assemble_step_operator(st, 1e-3, cache=cache)
u = torch.randn(op.layout.size, dtype=torch.float64, device="cuda")
out = torch.empty_like(u)
for _ in range(3):
    op.rows_device(u, False, out)
torch.cuda.synchronize()
