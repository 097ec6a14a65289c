"""Warm timeline of GMRES Arnoldi steps (torch.profiler / CUPTI, kernels as
they really overlap, unlike ncu's serialised cold-cache replay): per-kernel
busy time, GPU-busy union, idle gaps and the wall span of COUNT matvecs
starting at the START-th matvec of the second implicit step.
Usage: python tools/step_timeline.py c2|c4|c1 [START] [COUNT] [OUT.json]"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1602_05650_b200 import configs, solver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
start = int(sys.argv[2]) if len(sys.argv) > 2 else 20
count = int(sys.argv[3]) if len(sys.argv) > 3 else 10
out_path = sys.argv[4] if len(sys.argv) > 4 else None
st = {"c2": lambda: configs.aster(n_fibers=1024), "c4": lambda: configs.confined_aster(),
      "c1": lambda: configs.cloud_state("c1")}.get(cfg, lambda: configs.cloud_state(cfg))()
dt = 1e-3 if cfg in ("c2", "c4") else 5e-3
params = solver.GmresParams(tolerance=1e-8 if cfg == "c4" else 1e-10)
os.environ.setdefault("SF_GMRES_GRAPH", "0")   # GRAPH=1 replays captured Arnoldi steps
st, info = solver.backward_euler_step(st, dt, params, return_info=True)      # warm-up step

orig = solver.BlockOperator.rows_device
orig_prec = solver.Preconditioner.apply_device
calls = [0]
host = {"rows": 0.0, "prec": 0.0}
prof = profile(activities=[ProfilerActivity.CUDA])
marks = {}


def tick():
    calls[0] += 1
    if calls[0] == start:
        torch.cuda.synchronize()
        prof.start()
        marks["t0"] = time.perf_counter()
    elif calls[0] == start + count:
        torch.cuda.synchronize()
        marks["t1"] = time.perf_counter()
        prof.stop()


orig_graph_step = solver._ArnoldiGraph.step


def graph_step(self, vk, status):
    tick()
    return orig_graph_step(self, vk, status)


def rows(self, u, constants, out=None):
    if not constants:
        tick()
    h0 = time.perf_counter()
    r = orig(self, u, constants, out)
    if "t0" in marks and "t1" not in marks:
        host["rows"] += time.perf_counter() - h0
    return r


def prec(self, v, out=None):
    h0 = time.perf_counter()
    r = orig_prec(self, v, out)
    if "t0" in marks and "t1" not in marks:
        host["prec"] += time.perf_counter() - h0
    return r


solver.BlockOperator.rows_device = rows
solver.Preconditioner.apply_device = prec
solver._ArnoldiGraph.step = graph_step
torch.cuda.synchronize()
t0 = time.perf_counter()
st, info = solver.backward_euler_step(st, dt, params, return_info=True)
torch.cuda.synchronize()
el = time.perf_counter() - t0
solver.BlockOperator.rows_device = orig
solver.Preconditioner.apply_device = orig_prec

with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "trace.json")
    prof.export_chrome_trace(path)
    with open(path) as fh:
        trace = json.load(fh)
ev = [e for e in trace["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")
      and e.get("ph") == "X"]
ev.sort(key=lambda e: e["ts"])
span0 = ev[0]["ts"]
span1 = max(e["ts"] + e["dur"] for e in ev)
busy, cur0, cur1 = 0.0, None, None
gaps, big = [], []
last = None
for e in ev:
    a, b = e["ts"], e["ts"] + e["dur"]
    if cur1 is None or a > cur1:
        if cur1 is not None:
            busy += cur1 - cur0
            gaps.append(a - cur1)
            if a - cur1 > 5:
                big.append((round(a - cur1, 1), last["name"][:50], e["name"][:50]))
        cur0, cur1 = a, b
    else:
        cur1 = max(cur1, b)
    if last is None or b >= last["ts"] + last["dur"]:
        last = e
busy += cur1 - cur0
per = {}
streams = set()
for e in ev:
    k = e["name"][:90]
    r = per.setdefault(k, [0.0, 0])
    r[0] += e["dur"]
    r[1] += 1
    streams.add(e.get("args", {}).get("stream"))
rows_out = sorted(per.items(), key=lambda kv: -kv[1][0])
# the ordered launches of one period (from one sym_task_kernel start to the
# next: one Arnoldi step) with the idle time before each and its stream
syms = [i for i, e in enumerate(ev) if "sym_task_kernel" in e["name"]]
seq = []
if len(syms) >= 3:
    lo = ev[syms[1]]["ts"]
    prev_end = None
    for e in ev[syms[1]:syms[2] + 1]:
        gap = 0.0 if prev_end is None else max(0.0, e["ts"] - prev_end)
        seq.append((round(e["ts"] - lo, 1), round(e["dur"], 1), round(gap, 1),
                    e.get("args", {}).get("stream"), e["name"][:60]))
        end = e["ts"] + e["dur"]
        prev_end = end if prev_end is None else max(prev_end, end)
wall = 1e6 * (marks["t1"] - marks["t0"])
# steady-state period: start of the 2nd to start of the last symmetric (or,
# without one, pair) kernel of the window -- the first matvec carries the
# profiler's start-up gap
anchor = syms if len(syms) >= 3 else [i for i, e in enumerate(ev) if "pair_kernel" in e["name"]
                                      and "SbtP" in e["name"]]
period = ((ev[anchor[-1]]["ts"] - ev[anchor[1]]["ts"]) / (len(anchor) - 2)
          if len(anchor) >= 3 else None)
res = {"config": cfg, "step_ms": 1e3 * el, "iterations": info["iterations"],
       "matvecs": info["matvecs"], "window_matvecs": count,
       "wall_us_per_matvec": wall / count, "period_us": period,
       "gpu_span_us_per_matvec": (span1 - span0) / count,
       "gpu_busy_us_per_matvec": busy / count,
       "idle_gaps_us_per_matvec": sum(gaps) / count, "gaps_over_5us": sum(g > 5 for g in gaps),
       "streams": len(streams), "graph": os.environ["SF_GMRES_GRAPH"],
       "host_us_per_matvec": {k: 1e6 * v / count for k, v in host.items()},
       "kernels_us_per_matvec": {k: round(v[0] / count, 2) for k, v in rows_out},
       "launches_per_matvec": {k: v[1] / count for k, v in rows_out},
       "one_step_sequence": seq, "big_gaps": big}
print(f"{cfg}: steady Arnoldi-step period {period or 0:.1f} us")
print(f"{cfg}: step {1e3 * el:.1f} ms, {info['iterations']} its; window {count} matvecs: "
      f"wall {res['wall_us_per_matvec']:.1f} us, GPU span {res['gpu_span_us_per_matvec']:.1f}, "
      f"busy {res['gpu_busy_us_per_matvec']:.1f}, idle {res['idle_gaps_us_per_matvec']:.1f} us "
      f"per matvec ({res['gaps_over_5us']} gaps > 5 us, {len(streams)} streams); host enqueue "
      f"rows {res['host_us_per_matvec']['rows']:.0f} us, preconditioner "
      f"{res['host_us_per_matvec']['prec']:.0f} us per matvec (graph={res['graph']})")
for k, v in rows_out[:30]:
    print(f"  {v[0] / count:9.1f} us  x{v[1] / count:4.1f}  {k}")
print("idle gaps > 5 us (us, kernel before, kernel after):")
for g in big:
    print("  ", g)
print("one Arnoldi step: start_us dur_us idle_before_us stream kernel")
for r in seq:
    print("  %9.1f %8.1f %7.1f %6s  %s" % r)
if out_path:
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)
