"""Benchmark of the HI operator (one GMRES matvec's hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--mode fp64|fp32c]
    python bench.py --impl reference ...        # the reference's CPU path (oracle port)

A "step" is one application of the fiber HI operator to one batch of force
densities: the fused Stokeslet + (eps L)^2/2 doublet all-pairs sum over every
fiber node (complementary_velocities, system.py:623-709), the near-field
corrections and the local self terms M f + K_delta f (fiber.py:244-258).
Default workload: BASELINE config 5 (16,384 fibers x 64 nodes = 1,048,576
points, the largest single-GPU configuration), synthetic seeded inputs.
Multi-GPU: target-block sharding, NCCL all-gather of the force densities
once per step, fixed total work ("strong" scaling).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS_PER_PAIR = 35          # fused Stokeslet + doublet, minimal formula
# the symmetric kernel evaluates each unordered pair's geometry once: its own
# minimal work is 29 flops per directed interaction: per unordered pair the
# shared geometry r 3 + r^2 5 + rsqrt 1 + powers 3 = 12, per direction
# r.f 5 + a 2 + b 4 + accumulate 12 = 23; (12 + 2 x 23) / 2 = 29
FLOPS_PER_PAIR_SYM = 29
# FP64 hardware flops executed per interaction, from the ncu instruction
# counts of the symmetric kernel (DFMA x2 + DMUL + DADD per interaction,
# profiles/r01_ncu_counters.md: 12.52 x 2 + 5.01 + 1.54)
HW_FLOPS_PER_PAIR = 2 * 12.52 + 5.01 + 1.54
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--mode", default="fp64", choices=["fp64", "fp32c"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variant", action="store_true", help="skip the FP32c variant line")
    ap.add_argument("--launch-check", action="store_true",
                    help="start the ranks (gloo), print one JSON line per rank, do no work")
    ap.add_argument("--step-config", default="c1,c2,c2:body,c3,c4,c4:body,c4:body+ico,c5,c5:fp32c",
                    help="implicit-step workloads, comma separated, each with optional "
                         "':fp32c' / ':body' / ':warm' / ':ico' ('+'-joined) options ('' to skip)")
    ap.add_argument("--step-count", type=int, default=3, help="timed steps per small config")
    ap.add_argument("--big-step-count", type=int, default=1,
                    help="timed steps of c3/c4/c5 (2 s / 8 s / 38 s each on one GPU)")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks ----
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 7
                          for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------- reference (CPU) ----
_REF_KERNELS = None


def reference_kernels(threads):
    """slenderflow.kernels -- the reference's own numba kernels (staged in
    baseline/_ref by build()) with numba's prange over `threads` threads, or
    None when the reference is not staged."""
    global _REF_KERNELS
    if _REF_KERNELS is None:
        if not os.path.isdir(os.path.join(REF_PKG, "slenderflow")):
            _REF_KERNELS = False
        else:
            os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
            os.environ["NUMBA_NUM_THREADS"] = str(threads)
            import importlib
            sys.path.insert(0, REF_PKG)
            try:
                _REF_KERNELS = importlib.import_module("slenderflow.kernels")
            finally:
                sys.path.remove(REF_PKG)
    return _REF_KERNELS or None


def cpu_pair_rate(X, forces, eps, sample_rows, seed=0, use_reference=True):
    """The reference's pair sums on the host cores: the Stokeslet pass plus
    the doublet pass of complementary_velocities (system.py:656-671) for a
    row sample of targets against all sources, by slenderflow's OWN numba
    kernels (kernels.py:72-145, prange over every host thread; JIT compiled
    before timing) when the reference is staged, else by the oracle's C port
    of them (OpenMP).  Returns (pairs/s, seconds, pairs, threads, kind)."""
    from oracle import ops, pairs
    nf, n, _ = X.shape
    src = X.reshape(-1, 3)
    grp = np.repeat(np.arange(nf, dtype=np.int64), n)
    geos = [ops.geometry(X[m]) for m in range(nf)]
    w = np.concatenate([g["weights"] for g in geos])
    strengths = w[:, None] * forces.reshape(-1, 3)              # system.py:657-658
    c = np.repeat([(eps * g["L"]) ** 2 / 2.0 for g in geos], n)  # system.py:542
    dbl = c[:, None] * strengths
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(src.shape[0], size=sample_rows, replace=False))
    pref = 1.0 / (8.0 * np.pi)
    threads = host_threads()
    K = reference_kernels(threads) if use_reference else None
    if K is not None:
        t_src, t_grp = np.ascontiguousarray(src[rows]), np.ascontiguousarray(grp[rows])
        K.stokeslet_sum(t_src[:8], t_grp[:8], src[:64], grp[:64], strengths[:64], pref)   # JIT
        K.doublet_sum(t_src[:8], t_grp[:8], src[:64], grp[:64], dbl[:64], pref)
        t0 = time.perf_counter()
        u1, _ = K.stokeslet_sum(t_src, t_grp, src, grp, strengths, pref)
        u2, _ = K.doublet_sum(t_src, t_grp, src, grp, dbl, pref)
        dt = time.perf_counter() - t0
        kind = "reference"
    else:
        t0 = time.perf_counter()
        u1, _ = pairs.stokeslet_sum(src[rows], grp[rows], src, grp, strengths, pref)
        u2, _ = pairs.doublet_sum(src[rows], grp[rows], src, grp, dbl, pref)
        dt = time.perf_counter() - t0
        threads = pairs.num_threads()
        kind = "port"
    npairs = sample_rows * (src.shape[0] - n)
    return npairs / dt, dt, npairs, threads, kind


def workload_config(args, cloud, world):
    """The `config` object both arms report (same workload, same keys)."""
    return {"workload": f"{args.config}: HI operator matvec (Stokeslet+doublet all-pairs "
                        f"+ near + M+K_delta self terms), {cloud.n_fibers} fibers x "
                        f"{cloud.n_nodes} nodes",
            "points": cloud.n_points,
            "pairs_per_step": cloud.n_points ** 2 - cloud.n_fibers * cloud.n_nodes ** 2,
            "parallelism": f"target-shard{world}",
            "l2": "flushed between timed steps (256 MB write); K_delta 4.8 GB > L2"}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


REF_PKG = os.path.join(ROOT, "baseline", "_ref")


def c1_step_state(pkg):
    """C1 as implicit steps (the golden bstep_c1 case): 64 fibers, p = 31,
    centres in [-2,2]^3 with 2 eps L segment clearance (near pairs present,
    maps rebuilt every step), uniform force density (0,0,-1); built with
    `pkg`'s own constructors (this package's or slenderflow's)."""
    from paper_1602_05650_b200 import configs
    cl = configs.fiber_cloud(64, 31, eps=1e-2, E=1.0, region="cube", size=2.0, seed=0,
                             clear=2e-2, check="segment")
    fibs = [pkg["fiber"].Fiber(X, eps=1e-2, E=1.0) for X in cl.X]
    return pkg["system"].SystemState(
        fibs, force_models=[pkg["system"].UniformBodyForce(1.0, (0.0, 0.0, -1.0))])


def c2_step_state(pkg):
    """C2 (the golden bstep_c2 case): 1,024 fibers p = 31 clamped radially to
    an (8,8) sphere of radius 0.5, plus-end force 1 along the tangent."""
    from paper_1602_05650_b200 import configs
    pts, dirs = configs.aster_layout(1024, 0.5, 1.3, (0.0, 0.0, 0.0), 0.05, 0, "random")
    F, B = pkg["fiber"], pkg["body"]
    part = B.RigidParticle(B.make_surface(B.sphere_shape(0.5), (8, 8)))
    fibs = [F.straight_fiber(31, x0, d, 1.0, eps=1e-2, E=1.0,
                             bc_minus=F.ClampedToBody(0, x0, d),
                             bc_plus=F.PrescribedForceTorque(1.0 * d)) for x0, d in zip(pts, dirs)]
    return pkg["system"].SystemState(fibs, [part])


def reference_implicit_steps(threads, c2_iterations=None):
    """Implicit steps/s of the reference's OWN Python path -- slenderflow's
    backward_euler_step, unmodified, staged in baseline/_ref by build() --
    on the host cores (numba prange over `threads` threads, BLAS single
    threaded as SURVEY §6 prescribes, JIT compilation excluded).
    C1: one warm-up step, then two timed steps.  C2: a full step is ~7.5 min
    on 8 cores, so one step is timed in parts -- InteractionCache +
    assemble_step_operator + Preconditioner once, two matvecs
    (BlockOperator.apply + Preconditioner.apply) -- and the step is
    setup + (iterations + 2) matvecs with the reference's own iteration count
    (tests/golden/bstep_c2.npz), labelled as extrapolated."""
    if not os.path.isdir(os.path.join(REF_PKG, "slenderflow")):
        return {"unavailable": "reference not staged in baseline/_ref"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    os.environ["NUMBA_NUM_THREADS"] = str(threads)
    import importlib

    from threadpoolctl import threadpool_limits
    sys.path.insert(0, REF_PKG)
    try:
        pkg = {m: importlib.import_module(f"slenderflow.{m}")
               for m in ("fiber", "body", "system", "solver")}
    finally:
        sys.path.remove(REF_PKG)
    sv = pkg["solver"]
    out = []
    with threadpool_limits(1, user_api="blas"):
        st = c1_step_state(pkg)
        params = sv.GmresParams(tolerance=1e-10)
        sv.backward_euler_step(st, 5e-3, params)              # JIT warm-up
        times = []
        for _ in range(2):
            t0 = time.perf_counter()
            sv.backward_euler_step(st, 5e-3, params)
            times.append(time.perf_counter() - t0)
        out.append({"config": "c1: 64 fibers x 32 nodes cube cloud (near pairs), gravity",
                    "steps": 2, "ms_per_step": 1e3 * sum(times) / 2,
                    "steps_per_s": 2 / sum(times), "timing": "measured, full steps"})
        st = c2_step_state(pkg)
        t0 = time.perf_counter()
        cache = pkg["system"].InteractionCache(st)
        op, rhs = sv.assemble_step_operator(st, 1e-3, cache=cache)
        prec = sv.Preconditioner(op)
        setup = time.perf_counter() - t0
        u = np.random.default_rng(0).standard_normal(op.layout.size)
        mv = []
        for _ in range(2):
            t0 = time.perf_counter()
            prec.apply(op.apply(u))
            mv.append(time.perf_counter() - t0)
        its = c2_iterations
        if its is None:
            g = os.path.join(ROOT, "tests", "golden", "bstep_c2.npz")
            its = int(np.load(g)["iters_0"]) if os.path.exists(g) else 175
        step = setup + (its + 2) * min(mv)
        out.append({"config": "c2: 1024 fibers x 32 nodes clamped to a sphere (8x8 patches)",
                    "ms_per_step": 1e3 * step, "steps_per_s": 1.0 / step,
                    "setup_s": setup, "matvec_s": min(mv), "gmres_iterations": its,
                    "timing": "extrapolated: setup + (iterations + 2) x measured matvec"})
    return {"threads": threads, "steps": out}


def run_reference(args, rank, world):
    """The reference's pair sums on the host cores: slenderflow's own numba
    kernels (kernels.py:72-145, staged in baseline/_ref; the oracle C port if
    it is not staged), over every host thread.  A step is a bounded row
    sample of the config's matvec (each target row costs the same Ns pairs,
    SURVEY §8c), timed as it runs: ms_per_step is that sample's wall time,
    value its pair-interactions/s.  Plus slenderflow's own implicit steps
    (reference_implicit_steps)."""
    if rank != 0:
        return
    from oracle import pairs
    from paper_1602_05650_b200 import configs
    pairs.set_num_threads(host_threads())
    cloud = configs.make(args.config, seed=args.seed)
    f = configs.forces(cloud, seed=args.seed + 1)
    N = cloud.n_points
    rows = max(64, int(round(4e9 / N / 2)))  # ~4e9 pair evaluations (2 passes) per step
    rows = min(rows, N)
    for _ in range(args.warmup):
        cpu_pair_rate(cloud.X, f, cloud.eps, min(rows, 256), seed=1)
    rates, times = [], []
    for k in range(args.steps):
        r, dt, npairs, threads, kind = cpu_pair_rate(cloud.X, f, cloud.eps, rows, seed=100 + k)
        rates.append(r)
        times.append(dt)
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "stokes_pair_interactions_per_s", "value": value,
        "unit": "pair-interactions/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded rejection-sampled perturbed fiber cloud, N(0,1) forces)",
        "config": workload_config(args, cloud, world),
        "cpu_baseline": {"value": value, "unit": "pair-interactions/s", "cores": threads,
                         "kind": kind,
                         "sample": f"each step: {rows} target rows x {N} sources, Stokeslet + "
                                   f"doublet passes ("
                                   + ("slenderflow.kernels, the reference's own numba kernels, "
                                      "prange" if kind == "reference" else
                                      "oracle/oracle_pairs.c, the C port, OpenMP")
                                   + f" on {threads} host threads); ms_per_step is the sample's "
                                   f"own wall time (a full matvec is {N / rows:.0f}x the sample)"},
        "e2e": {"value": value, "unit": "pair-interactions/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "implicit_steps": (reference_implicit_steps(threads)
                           if args.step_config else None),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------- implicit steps ----
def measure_steps(config, count, comm=None, warm=True):
    """Implicit steps/s of the full device step (cache, self blocks, block LU,
    GMRES to tol 1e-10, state update) on BASELINE config 2 (1024-fiber aster)
    or a sedimenting cloud; one warm-up step, then `count` timed steps."""
    import torch

    from paper_1602_05650_b200 import configs, solver
    config, _, opts = config.partition(":")
    opts = set(opts.split("+")) if opts else set()
    precision = "fp32c" if "fp32c" in opts else "fp64"
    body = "body" in opts          # body-coupled preconditioner (not in the reference)
    warm_start = "warm" in opts    # GMRES warm start from the current state (not in the reference)
    from paper_1602_05650_b200 import body as body_, fiber as fiber_, system as system_
    ours = {"fiber": fiber_, "body": body_, "system": system_}
    if config == "c1":
        st = c1_step_state(ours)
        dt, tol = 5e-3, 1e-10
        desc = "c1: 64 fibers x 32 nodes cube cloud (near pairs), gravity"
    elif config == "c2":
        st = c2_step_state(ours)
        dt, tol = 1e-3, 1e-10
        desc = "c2: 1024 fibers x 32 nodes clamped to a sphere (8x8 patches), plus-end force 1"
    elif config == "c4":
        ico = "ico" in opts
        st = configs.confined_aster(periphery_mesh="ico" if ico else "patch")
        dt, tol = 1e-3, 1e-8
        desc = ("c4: 2048 fibers x 32 nodes clamped to a centrosome in a "
                + ("40,962-vertex icosphere periphery (BASELINE's literal mesh; beyond the "
                   "reference)" if ico else "40,960-node periphery")
                + ", fiber<->boundary and boundary<->boundary double layers")
    else:
        st = configs.cloud_state(config)
        dt, tol = 5e-3, 1e-10
        desc = f"{config}: sedimenting cloud, {len(st.fibers)} fibers"
    params = solver.GmresParams(tolerance=tol)
    if comm is None:
        def one(st):
            return solver.backward_euler_step(st, dt, params, return_info=True,
                                              precision=precision, body_coupling=body,
                                              warm_start=warm_start)
    else:
        from paper_1602_05650_b200 import dsolver

        if warm_start:
            raise ValueError("warm start is a single-GPU option")

        def one(st):
            return dsolver.dist_backward_euler_step(st, dt, comm, params, return_info=True,
                                                    precision=precision, body_coupling=body)

    def sync():
        torch.cuda.synchronize()
        if comm is not None:
            import torch.distributed as dist
            dist.barrier()
    if warm:
        st, info = one(st)
    times, iters = [], []
    for _ in range(count):
        sync()
        t0 = time.perf_counter()
        st, info = one(st)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        iters.append(info["iterations"])
    if comm is not None:                       # max over ranks, per step
        t = torch.tensor(times, dtype=torch.float64, device="cuda")
        comm.dist.all_reduce(t, op=comm.dist.ReduceOp.MAX)
        times = t.tolist()
    return {"config": desc, "precision": precision,
            "preconditioner": ("body-coupled (not in the reference)" if body
                               else "block Jacobi (reference)"),
            "initial_guess": ("current state (not in the reference)" if warm_start
                              else "zero (reference)"),
            "dt": dt, "gmres_tol": tol, "steps": count,
            "ranks": 1 if comm is None else comm.world,
            "steps_per_s": count / sum(times), "ms_per_step": 1e3 * sum(times) / count,
            "gmres_iterations": iters,
            "timing": "wall clock around each full step (host orchestration included), "
                      + ("after one warm-up step" if warm else
                         "no warm-up step of its own (the preceding step runs warmed the path)")
                      + "; max over ranks"}


# ---------------------------------------------------------------- ours (GPU) ----
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1602_05650_b200 import _native, configs, kernels
    from paper_1602_05650_b200.dist import ShardedHIOperator
    from paper_1602_05650_b200.operator import FiberHIOperator

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    _native.load(require_device=True)
    mode = _native.SF_MODE_FP64 if args.mode == "fp64" else _native.SF_MODE_FP32C
    cloud = configs.make(args.config, seed=args.seed)
    f_all = configs.forces(cloud, seed=args.seed + 1)
    # the reference's state and interaction cache for this cloud: its near-field
    # maps (system.py:564-599; C5 has 2 targets inside another fiber's near
    # shell) complete the operator, and it serves the reference-API e2e below
    from paper_1602_05650_b200 import system as sysm
    from paper_1602_05650_b200.fiber import Fiber
    st_api = sysm.SystemState([Fiber(X, eps=cloud.eps, E=cloud.E) for X in cloud.X])
    cache = sysm.InteractionCache(st_api, device=dev)
    near = cache.near_fiber
    op = FiberHIOperator(cloud.X, cloud.eps, device=dev, mode=mode, shard=(rank, world),
                         near=near)
    sop = ShardedHIOperator(op)
    f_local = torch.as_tensor(f_all[op.f0:op.f0 + op.nown], device=dev).contiguous()
    u_nl = torch.empty((op.Nown, 3), dtype=torch.float64, device=dev)
    u_self = torch.empty((op.Nown, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2

    def step():
        sop.apply(f_local, out_nl=u_nl, out_self=u_self)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    op.check_bad()
    barrier()
    # ---- timed region: exactly K steps, L2 flushed between steps (outside events)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        barrier()
        for k in range(args.steps):
            flush.fill_(float(k))
            starts[k].record()
            step()
            ends[k].record()
        barrier()
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_step = sum(ms) / len(ms)
    t = torch.tensor([ms_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    total_pairs = cloud.n_points ** 2 - cloud.n_fibers * cloud.n_nodes ** 2
    value = total_pairs / (ms_step * 1e-3)

    # ---- e2e: host (pinned) forces in, host velocities out, through the public API
    f_host = torch.as_tensor(f_all[op.f0:op.f0 + op.nown]).pin_memory()
    out_host = torch.empty((2, op.Nown, 3), dtype=torch.float64).pin_memory()
    e_s = torch.cuda.Event(enable_timing=True)
    e_e = torch.cuda.Event(enable_timing=True)
    barrier()
    e_s.record()
    for _ in range(args.steps):
        fd = f_host.to(dev, non_blocking=True)
        a, b = sop.apply(fd)
        out_host[0].copy_(a, non_blocking=True)
        out_host[1].copy_(b, non_blocking=True)
    e_e.record()
    barrier()
    e2e_ms = torch.tensor([e_s.elapsed_time(e_e) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # ---- roofline of the dominant kernel (pack + pair + ordered reduce), this GPU
    reps = max(2, min(args.steps, 3))
    fs = sop.gather_sources(f_local)
    r_s = torch.cuda.Event(enable_timing=True)
    r_e = torch.cuda.Event(enable_timing=True)
    if op.symmetric_shard:       # N > 1: this rank's share of the unit-pair tasks
        part = torch.empty((op.N, 3), dtype=torch.float64, device=dev)

        def dominant():
            op.symmetric_partial(fs, out=part)
        rank_pairs = op.shard_pairs
    else:
        def dominant():
            op.apply(fs, out_nl=u_nl, self_terms=False)
        rank_pairs = op.pairs_per_apply
    dominant()
    torch.cuda.synchronize()
    r_s.record()
    for _ in range(reps):
        dominant()
    r_e.record()
    torch.cuda.synchronize()
    pair_ms = r_s.elapsed_time(r_e) / reps
    peak_flops, _ = kernels.dfma_peak(1 << 15)
    achieved = rank_pairs * FLOPS_PER_PAIR / (pair_ms * 1e-3)
    traffic = None
    traffic_wave = None
    prof = os.path.join(ROOT, "profiles", "r02_ncu_sym_c5_wave_metrics.json")
    if args.config == "c5" and world == 1 and op.symmetric and os.path.exists(prof):
        # ncu --set full of one wave launch of the task kernel; scaled to the
        # matvec by the number of wave launches (all but the last are full)
        m = json.load(open(prof))
        gb = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        traffic_wave = sum(float(m[k][1].replace(",", "")) * gb.get(m[k][0], 1.0)
                           for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
        n_waves = (_native.load().sf_sym_launch_count(op.N, op.n, op.mode, 0, 1) - 3) // 2
        traffic = traffic_wave * n_waves

    # ---- the FP32-compute / FP64-accumulate variant on the same workload
    variant = None
    if args.mode == "fp64" and not args.no_variant:
        op32 = FiberHIOperator(cloud.X, cloud.eps, device=dev, mode=_native.SF_MODE_FP32C,
                               shard=(rank, world), near=near)
        sop32 = ShardedHIOperator(op32)
        u32 = torch.empty_like(u_nl)
        for _ in range(2):
            sop32.apply(f_local, out_nl=u32, out_self=u_self)
        barrier()
        v_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        v_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for k in range(args.steps):
            flush.fill_(float(k))
            v_s[k].record()
            sop32.apply(f_local, out_nl=u32, out_self=u_self)
            v_e[k].record()
        barrier()
        vms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(v_s, v_e)) / args.steps],
                           dtype=torch.float64, device=dev)
        sop.apply(f_local, out_nl=u_nl, out_self=u_self)            # FP64 reference rows
        err = torch.stack([((u32 - u_nl) ** 2).sum(), (u_nl ** 2).sum()])
        if world > 1:
            dist.all_reduce(vms, op=dist.ReduceOp.MAX)
            dist.all_reduce(err)
        vms = float(vms.item())
        variant = {"dtype": "f32-compute/f64-accumulate", "value": total_pairs / (vms * 1e-3),
                   "unit": "pair-interactions/s", "ms_per_step": vms,
                   "rel_l2_vs_fp64": float((err[0] / err[1]).sqrt().item()),
                   "tolerance": 1e-5,
                   # whole matvec (self terms included), against the NOMINAL FP32 peak
                   # of 148 SMs x 128 lanes x 2 x 1.965 GHz: there is no measured FP32
                   # figure in MEASURED_PEAKS.json (profiles/r02_ffma2_probe2.txt
                   # measures 73.3 TFLOP/s with packed FFMA2)
                   "roofline": {"bound": "fp32", "unit": "TFLOP/s", "flops_per_pair": 35,
                                "achieved": 35.0 * total_pairs / (vms * 1e-3) / 1e12 / world,
                                "peak": 74.4, "peak_source": "nominal",
                                "frac": 35.0 * total_pairs / (vms * 1e-3) / 1e12 / world / 74.4}}
        del op32, sop32, u32

    # ---- e2e through the reference's own operator signature (world 1):
    # system.complementary_velocities(state, fiber_forces=[per-fiber numpy
    # arrays], cache=cache) -> per-fiber numpy velocities (system.py:623-709)
    ref_api = None
    if world == 1 and args.mode == "fp64":
        f_list = [f_all[m] for m in range(cloud.n_fibers)]
        res = sysm.complementary_velocities(st_api, fiber_forces=f_list, cache=cache)
        u_api = np.concatenate(res.fibers)
        api_rel = float(np.linalg.norm(u_api - u_nl.cpu().numpy()) / np.linalg.norm(u_api))
        t_api = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sysm.complementary_velocities(st_api, fiber_forces=f_list, cache=cache)
            t_api.append(time.perf_counter() - t0)
        ms_api = 1e3 * sum(t_api) / len(t_api)
        ref_api = {"value": total_pairs / (ms_api * 1e-3), "unit": "pair-interactions/s",
                   "ms_per_step": ms_api,
                   "call": "system.complementary_velocities(state, fiber_forces=[16384 (64,3) "
                           "numpy arrays], cache=InteractionCache(state)) -> per-fiber numpy "
                           "velocities; the non-local part only (no self terms), host wall clock",
                   "h2d_bytes_per_step": int(cloud.n_points * 3 * 8),
                   "d2h_bytes_per_step": int(cloud.n_points * 3 * 8),
                   "rel_diff_vs_operator_nonlocal": api_rel}
    del cache, st_api

    steps = []
    if args.step_config:
        from paper_1602_05650_b200.dsolver import TorchComm
        comm = TorchComm() if world > 1 else None
        cfgs = [c for c in args.step_config.split(",") if c]
        if comm is not None:           # the warm start is single-GPU only
            cfgs = [c for c in cfgs if "warm" not in c.partition(":")[2].split("+")]
        for k, cfg in enumerate(cfgs):
            big = cfg.split(":")[0] in ("c3", "c4", "c5")
            try:
                steps.append(measure_steps(cfg, args.big_step_count if big else args.step_count,
                                           comm, warm=not (big and k > 0)))
            except Exception as err:      # noqa: BLE001 - reported in the JSON line
                steps.append({"config": cfg, "error": f"{type(err).__name__}: {err}"})

    lines = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            pairs_mod_threads = host_threads()
            from oracle import pairs as _pairs
            _pairs.set_num_threads(pairs_mod_threads)
            rows = max(64, int(round(2e10 / cloud.n_points)))     # ~13 s on 16 host cores
            rate, dt, npairs, threads, kind = cpu_pair_rate(cloud.X, f_all, cloud.eps, rows)
            cpu = {"value": rate, "unit": "pair-interactions/s", "cores": threads, "kind": kind,
                   "sample": f"{rows} target rows x {cloud.n_points} sources, Stokeslet + doublet "
                             f"passes of "
                             + ("slenderflow's own numba kernels" if kind == "reference"
                                else "the oracle C port (OpenMP)") + f", {dt:.1f} s"}
        clocks = clk.summary()
        lines = {
            "metric": "stokes_pair_interactions_per_s", "value": value,
            "unit": "pair-interactions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.mode == "fp64" else "f32-compute/f64-accumulate",
            "data": "synthetic (seeded rejection-sampled perturbed fiber cloud, N(0,1) forces)",
            "config": workload_config(args, cloud, world),
            "matvecs_per_s": 1e3 / ms_step, "near_maps": len(near),
            "roofline": {"bound": "fp64", "achieved": achieved / 1e12,
                         "peak": peak_flops / 1e12, "unit": "TFLOP/s",
                         "frac": achieved / peak_flops, "traffic": traffic,
                         "frac_alg_sym": rank_pairs * FLOPS_PER_PAIR_SYM / (pair_ms * 1e-3)
                         / peak_flops,
                         "frac_hw": rank_pairs * HW_FLOPS_PER_PAIR / (pair_ms * 1e-3) / peak_flops,
                         "frac_note": "frac: 35-flop one-sided convention (SURVEY §8d); "
                                      "frac_alg_sym: 29 flops per directed interaction, the "
                                      "symmetric kernel's own minimal work; frac_hw: FP64 "
                                      "hardware flops executed per interaction (ncu "
                                      "instruction counts)",
                         "traffic_wave": traffic_wave,
                         "traffic_note": "DRAM bytes of the task kernel per matvec, like "
                                         "achieved: ncu bytes of one wave launch "
                                         "(traffic_wave, profiles/r02_ncu_sym_c5_wave_metrics"
                                         ".json) x the wave launches of one matvec; mostly "
                                         "the wave's partial sums (written once, read once by "
                                         "the ordered reduce) and source re-reads after they "
                                         "evict the 80 MB of packed sources from L2; the "
                                         "kernel is FP64-pipe bound (7 GB/s of DRAM), not "
                                         "HBM bound",
                         "kernel": "pack + slab meta + sym_task_kernel (symmetric fiber-fiber "
                                   "pairs) + ordered partial reduce",
                         "flops_per_pair": FLOPS_PER_PAIR,
                         "peak_source": "measured DFMA microbenchmark (sf_dfma_peak) on this GPU; "
                                        f"nominal {NOMINAL_FP64_TFLOPS:.1f} TFLOP/s at 1965 MHz",
                         "kernel_ms": pair_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": total_pairs / (e2e_ms * 1e-3), "unit": "pair-interactions/s",
                    "h2d_bytes_per_step": int(cloud.n_points * 3 * 8),
                    "d2h_bytes_per_step": int(2 * cloud.n_points * 3 * 8)},
            "gpu_launches": args.steps * op.launches_per_apply,
            "clocks": clocks,
            "variant_fp32c": variant,
            "e2e_reference_api": ref_api,
            "implicit_steps": steps,
        }
        print(json.dumps(lines), flush=True)
    barrier()


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """`bench.py --gpus N` (N > 1) without a torchrun environment: launch the
    N ranks here, one process per GPU, exactly as the driver's torchrun
    command would (127.0.0.1 rendezvous), and return their exit code.  Never
    silently measures fewer ranks than asked for."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def init_ranks(args, rank, world, local_rank):
    """Process group for world > 1; checks that the world matches --gpus and
    that every rank has its own GPU (NCCL), failing loudly otherwise."""
    import torch
    import torch.distributed as dist
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # SF_DIST_BACKEND=gloo: functional check of the multi-rank code path with
    # host-side collectives (never a scaling number); ranks may share a GPU
    backend = os.environ.get("SF_DIST_BACKEND", "nccl")
    if args.launch_check:
        backend = "gloo"
    elif backend == "nccl" and torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, "
                         f"found {torch.cuda.device_count()}")
    if backend == "nccl":
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        if torch.cuda.is_available():
            local_rank = local_rank % torch.cuda.device_count()
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
    return local_rank


def main():
    args = parse()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        run_reference(args, rank, world)
        return
    if world > 1:
        local_rank = init_ranks(args, rank, world, local_rank)
    try:
        if args.launch_check:          # launcher test: report the rank layout, no work
            # one write(2) per rank so the lines of concurrent ranks never interleave
            line = json.dumps({"launch_check": True, "rank": rank, "world": world,
                               "local_rank": local_rank}) + "\n"
            sys.stdout.flush()
            os.write(sys.stdout.fileno(), line.encode())
            return
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
