"""bench.py's launcher (CPU, no GPU needed): `--gpus N` without a torchrun
environment starts N ranks itself, and a world that disagrees with --gpus
fails loudly instead of measuring fewer ranks."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


def test_gpus_two_self_launches_two_ranks():
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--launch-check"], cwd=ROOT,
                         env=_env(), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)


def test_world_mismatch_fails_loudly():
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--launch-check"], cwd=ROOT,
                         env=_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0",
                                  MASTER_ADDR="127.0.0.1", MASTER_PORT="29611"),
                         capture_output=True, text=True, timeout=600)
    assert out.returncode != 0
    assert "WORLD_SIZE=2" in out.stderr
