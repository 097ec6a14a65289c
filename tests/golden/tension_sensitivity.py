"""How well FP64 determines the implicit-step trajectory at the BASELINE
orders, measured on the REFERENCE itself (build container only):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        OPENBLAS_NUM_THREADS=1 python tests/golden/tension_sensitivity.py [case[:steps] ...]

For each make_golden_baseline case, slenderflow runs the first steps twice:
from the fixture's initial centrelines and from the same centrelines times
(1 + 1e-15 xi), xi ~ N(0,1) (a perturbation at the level of FP64 rounding).
The relative change of X, T, U, q1 and q0 after every step is written to
tension_sensitivity.json ("dX", "dT", ... for the first step, "steps"
with one record per step, and "operator": the change of the first step's
A u, rhs and M v).  At p = 31 the inextensibility rows are sums of
D_s^4 terms of size ~1e12 that cancel to O(1), so T (and the surface
densities, which balance the clamped fibers' end loads) move by 1e-4-1e-3
under rounding-level input changes while X moves by ~1e-10: any FP64
implementation with another summation order (this one included) can match
the reference's T and q only to that level."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import make_golden_baseline as mg  # noqa: E402
from slenderflow import solver  # noqa: E402


def run(case, nsteps, scale=None):
    st, inputs, spec, dt, tol, _ = mg.CASES[case]()
    if scale is not None:
        for f, s in zip(st.fibers, scale):
            f.X = f.X * s
    out = []
    for _ in range(nsteps):
        solver.backward_euler_step(st, dt, solver.GmresParams(tolerance=tol))
        rec = dict(X=np.stack([f.X for f in st.fibers]), T=np.stack([f.T for f in st.fibers]))
        if st.particles:
            rec["U"] = np.stack([p.U for p in st.particles])
            rec["q1"] = np.stack([p.q for p in st.particles])
        if st.periphery is not None:
            rec["q0"] = np.asarray(st.periphery.q)
        out.append(rec)
    return out


def operator_records(case, scale=None):
    """A u, rhs and M v of the first step (the seeded u, v of the fixture)."""
    st, inputs, spec, dt, tol, _ = mg.CASES[case]()
    if scale is not None:
        for f, s in zip(st.fibers, scale):
            f.X = f.X * s
    op, rhs = solver.assemble_step_operator(st, dt)
    n = op.layout.size
    u = np.random.default_rng(mg.SEED_U).standard_normal(n)
    v = np.random.default_rng(mg.SEED_V).standard_normal(n)
    return dict(Au=op.apply(u), rhs=rhs, Mv=solver.Preconditioner(op).apply(v))


def rel(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / d) if d else float(np.linalg.norm(a))


def main(specs):
    path = os.path.join(HERE, "tension_sensitivity.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for spec in specs:
        case, _, ns = spec.partition(":")
        ns = int(ns or 1)
        st0, *_ = mg.CASES[case]()
        X0 = np.stack([f.X for f in st0.fibers])
        xi = np.random.default_rng(0).standard_normal(X0.shape)
        a = run(case, ns)
        b = run(case, ns, scale=1.0 + 1e-15 * xi)
        steps = [{k: rel(rb[k], ra[k]) for k in ra} for ra, rb in zip(a, b)]
        oa, ob = operator_records(case), operator_records(case, scale=1.0 + 1e-15 * xi)
        ops = {k: rel(ob[k], oa[k]) for k in oa}
        out[case] = dict(perturbation=1e-15, **{"d" + k: v for k, v in steps[0].items()},
                         steps=steps, operator=ops)
        print(case, steps, flush=True)
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["bstep_c1:10", "bstep_aster256:3", "bstep_confined:2"])
