"""Implicit-step wall time: single-GPU solver vs the distributed solver
(dsolver) under torchrun (NCCL).  Usage:
  torchrun --nproc-per-node 1 --master-addr 127.0.0.1 tools/dist_step_perf.py [config]"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1602_05650_b200.dsolver import TorchComm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
lr = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(lr)
dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
comm = TorchComm()
d = bench.measure_steps(cfg, 2, comm)
if comm.rank == 0:
    print("dist  ", d["ms_per_step"], d["gmres_iterations"], flush=True)
if comm.world == 1:
    s = bench.measure_steps(cfg, 2, None)
    print("single", s["ms_per_step"], s["gmres_iterations"], flush=True)
dist.destroy_process_group()
