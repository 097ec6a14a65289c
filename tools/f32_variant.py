"""FP32-compute variant of the symmetric fiber-pair kernel at full C5 size:
pair-interactions/s (CUDA events, L2 flushed) and rel L2 against FP64, for
the kernel variant selected by SF_SYM_F32_VARIANT (34: scalar FFMA, 134:
packed FFMA2 with 3 CTAs/SM, 124: packed with 2 CTAs/SM)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_1602_05650_b200 import _native, configs  # noqa: E402
from paper_1602_05650_b200.operator import FiberHIOperator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
cl = configs.make(cfg, seed=0)
f = torch.as_tensor(configs.forces(cl, seed=1), device="cuda")
op64 = FiberHIOperator(cl.X, cl.eps, device="cuda")
op32 = FiberHIOperator(cl.X, cl.eps, device="cuda", mode=_native.SF_MODE_FP32C)
u64, _ = op64.apply(f, self_terms=False)
u64 = u64.clone()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
u32, _ = op32.apply(f, self_terms=False)
ms = []
for k in range(3):
    flush.fill_(float(k))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    u32, _ = op32.apply(f, self_terms=False)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
pairs = cl.n_points ** 2 - cl.n_fibers * cl.n_nodes ** 2
t = min(ms)
print(json.dumps({"config": cfg, "variant": os.environ.get("SF_SYM_F32_VARIANT", "default"),
                  "ms": t, "pairs_per_s": pairs / (t * 1e-3),
                  "rel_l2_vs_fp64": float((u32 - u64).norm() / u64.norm())}), flush=True)
