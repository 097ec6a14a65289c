"""Time the symmetric fiber x fiber sum on the C2 aster geometry (1024 fibers
x 32 nodes clamped around a sphere), the densest-core case for slab boxes.
Tuning helper: SF_SYM_VARIANT / SF_SYM_UNIT select the launch shape."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_05650_b200 import configs  # noqa: E402
from paper_1602_05650_b200.operator import FiberHIOperator  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
st = configs.aster(n_fibers=nf)
X = np.stack([f.X for f in st.fibers])
F = np.random.default_rng(1).standard_normal(X.shape)
op = FiberHIOperator(X, 1e-2)
f = torch.as_tensor(F, device="cuda")
u = torch.empty((op.N, 3), dtype=torch.float64, device="cuda")
for _ in range(3):
    op.apply(f, out_nl=u, self_terms=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
s.record()
for _ in range(reps):
    op.apply(f, out_nl=u, self_terms=False)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
print(json.dumps({"fibers": nf, "variant": os.environ.get("SF_SYM_VARIANT", "default"),
                  "unit": os.environ.get("SF_SYM_UNIT", "auto"), "ms": ms,
                  "gpairs_s": op.pairs_per_apply / ms / 1e6}))
