#!/usr/bin/env python
"""BASELINE config 2 on the GPU path: manufactured-solution convergence sweep.

    python scripts/convergence.py [--N 1 2 ... 7] [--n 4 8 16] [--T 0.5] [--out profiles/convergence_r1.json]
    python scripts/convergence.py --study wavespeed      (N=6, k = 1/4/8/12, M = 0..6)

Kuhn meshes of n^3 cubes (384 / 3072 / 24576 tets), N = 1..7, M = N, smooth c^2 = 1 + 1/2 sin sin sin,
manufactured solution with source (reading R17), T = 0.5, dt = 0.5 h_min / (c_max (N+1)^2)
(R14).  Reports ||p_h(T) - p(T)||_{L2} (R18) and the observed rates; the paper predicts
r = min(N+1, M+3) = N+1 for M = N.  Every step runs in libbbwadg.so (bbwadg_run).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


_CACHE = {}


def run_case(N, n, T, dtype="f64", M=None, k=1.0):
    """Input synthesis (L2 fits) runs with torch on the GPU; the initial state and the source are cached
    per (N, n) and (N, n, k)."""
    from paper_1808_08645_b200 import Solver
    from workloads import errors, kuhn, media, states

    M = N if M is None else M
    dev = "cuda"
    if ("mesh", n) not in _CACHE:
        _CACHE[("mesh", n)] = kuhn.kuhn_mesh(n)
    v, e = _CACHE[("mesh", n)]
    f = media.c2_smooth(k)
    c2 = media.project_c2(v, e, f, M, device=dev)
    if ("q0", N, n) not in _CACHE:
        _CACHE[("q0", N, n)] = states.manufactured_initial(v, e, N, device=dev)
    if ("src", N, n, k) not in _CACHE:
        _CACHE[("src", N, n, k)] = states.manufactured_source(v, e, N, f, device=dev)
    s = Solver(v, e, N, M, c2, dtype=dtype)
    s.set_source(_CACHE[("src", N, n, k)])
    s.set_state(_CACHE[("q0", N, n)])
    dt0 = 0.5 * kuhn.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
    nst = int(np.ceil(T / dt0))
    t0 = time.perf_counter()
    s.run(0.0, T / nst, nst)
    s.synchronize()
    el = time.perf_counter() - t0
    Q = np.asarray(s.get_state(), dtype=np.float64)
    s.close()
    err = errors.l2_error(v, e, Q[:, 0], N, lambda x, y, z: states.manufactured_exact(x, y, z, T)[0])
    return {"N": N, "M": M, "k": k, "n": n, "K": int(len(e)), "steps": nst, "err_p": err, "gpu_seconds": el}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, nargs="+", default=list(range(1, 8)))
    ap.add_argument("--n", type=int, nargs="+", default=[4, 8, 16])
    ap.add_argument("--T", type=float, default=0.5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--study", choices=["refinement", "wavespeed", "mlessn"], default="refinement")
    a = ap.parse_args()
    if a.study == "mlessn":
        # P:678 / Fig. con3d: N = 4 and 5, M = 0, 1, 2 < N; observed rate r = 2 for M = 0 and
        # r = min(N+1, M+3) for M >= 1 (4 for M = 1, 5 for N = 4 / M = 2); smooth c^2 (k = 1) as in the paper
        rows = []
        for N in (4, 5):
            for M in (0, 1, 2):
                prev = None
                for n in a.n:
                    r = run_case(N, n, a.T, M=M)
                    r["rate"] = None if prev is None else float(np.log2(prev / r["err_p"]))
                    r["predicted_rate"] = 2 if M == 0 else min(N + 1, M + 3)
                    prev = r["err_p"]
                    rows.append(r)
                    print(json.dumps(r), flush=True)
        out = {"study": "P:678 M < N convergence (3D): N = 4, 5; M = 0, 1, 2; Kuhn meshes n = %s, T = %g" % (a.n, a.T),
               "predicted_rate": "2 for M = 0, min(N+1, M+3) for M >= 1 (P:678)", "rows": rows}
        with open(a.out or os.path.join(ROOT, "profiles", "convergence_mlessn_r2.json"), "w") as fh:
            json.dump(out, fh, indent=1)
        return
    if a.study == "wavespeed":
        # P:1048-1251 (Fig. wavespeed, 3D): N = 6, uniform mesh h = 0.0833 (n = 24 cubes on [-1,1]^3,
        # 82,944 tets), c^2 = 1 + 1/2 sin(k pi x) sin(k pi y) sin(k pi z), k = 1, 4, 8, 12, M = 0..N;
        # the manufactured solution is the same for every k (its source carries c^2).
        rows = []
        for k in (1.0, 4.0, 8.0, 12.0):
            for M in range(0, 7):
                r = run_case(6, 24, a.T, M=M, k=k)
                rows.append(r)
                print(json.dumps(r), flush=True)
        out = {"study": "P:1048-1251 wavespeed frequency study (3D): N=6, n=24 (h=1/12), T=%g" % a.T,
               "expected": "error grows with k at fixed M and falls with M (P:1251)", "rows": rows}
        with open(a.out or os.path.join(ROOT, "profiles", "wavespeed_r1.json"), "w") as fh:
            json.dump(out, fh, indent=1)
        return
    rows = []
    for N in a.N:
        prev = None
        for n in a.n:
            r = run_case(N, n, a.T)
            r["rate"] = None if prev is None else float(np.log2(prev / r["err_p"]))
            prev = r["err_p"]
            rows.append(r)
            print(json.dumps(r), flush=True)
    out = {"study": "BASELINE config 2: manufactured solution, M = N, T = %g, Kuhn meshes n = %s" % (a.T, a.n),
           "predicted_rate": "N+1 (P:678, r = min(N+1, M+3))", "rows": rows}
    with open(a.out or os.path.join(ROOT, "profiles", "convergence_r1.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
