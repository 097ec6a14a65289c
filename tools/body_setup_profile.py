"""Where does the body-coupled preconditioner's setup go? (C2 / C4)"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
st = configs.aster(n_fibers=1024) if cfg == "c2" else configs.confined_aster()
op, rhs = solver.assemble_step_operator(st, 1e-3)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op._pcache = None
    p0 = solver.Preconditioner(op)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    p1 = solver.Preconditioner(op, body_coupling=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    B = op.particle_block_matrix()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    op._pcache = None
    y = torch.zeros(op.layout.size, dtype=torch.float64, device=op.device)
    op.particle_rows_device(y)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    op.particle_rows_device(y)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    LU = torch.linalg.inv_ex(B)
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    v = torch.randn(op.layout.size, dtype=torch.float64, device=op.device)
    p1.apply_device(v)
    torch.cuda.synchronize()
    t7 = time.perf_counter()
    p0.apply_device(v)
    torch.cuda.synchronize()
    t8 = time.perf_counter()
    print(f"{cfg} rep {rep}: block-Jacobi setup {1e3*(t1-t0):.1f} ms, coupled setup {1e3*(t2-t1):.1f} ms "
          f"[particle block {1e3*(t3-t2):.1f}, particle cache+rows {1e3*(t4-t3):.1f}, rows {1e3*(t5-t4):.2f}, "
          f"LU {1e3*(t6-t5):.1f}]; apply coupled {1e3*(t7-t6):.2f} ms vs bj {1e3*(t8-t7):.2f} ms",
          flush=True)
