"""bench.py's multi-rank path (the driver's N > 1 launch) run end to end on
one GPU: torchrun with 2 ranks and host-side (gloo) collectives, so no kernel
waits on another rank's kernel.  Checks the JSON contract of rank 0's line
and that rank 1 prints nothing."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_gloo(cuda):
    env = dict(os.environ, SF_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
           "--config", "c3_scaled", "--steps", "1", "--warmup", "1", "--no-cpu-baseline",
           "--step-config", "c2,c2:body", "--step-count", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                      # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["parallelism"] == "target-shard2"
    assert d["variant_fp32c"]["rel_l2_vs_fp64"] < 1e-5
    steps = d["implicit_steps"]
    assert len(steps) == 2 and all(s["ranks"] == 2 for s in steps)
    assert steps[1]["preconditioner"].startswith("body-coupled")   # distributed body coupling
    assert steps[1]["gmres_iterations"][0] < steps[0]["gmres_iterations"][0]
    assert "error" not in steps[0] and steps[0]["gmres_iterations"][0] > 0
