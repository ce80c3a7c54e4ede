"""GPU accuracy studies for the round-2 rows (NEXT-2 elastic, NEXT-4 2D), through the C ABI:

* 2D: the paper's 2D manufactured solution on n x n x 2 triangle meshes, N = 4, 5 and M = 0..3 -- the
  Fig. con2d experiment on our square meshes (rates transfer, constants do not; P:678 predicts r = 2 for
  M = 0 and min(N+1, M+3) for M >= 1);
* elastic: the exact standing P-wave of DESIGN.md R27 (lambda = 0, mu = 1/2, rho = 1, traction-free box), N = 2..5,
  M = 1, rate N+1 expected.
Error norms by the oracles' l2_error (quadrature only).   python scripts/convergence_new_rows.py OUT.json
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.acoustic2d import Acoustic2DOracle  # noqa: E402
from oracle.elastic import ElasticOracle  # noqa: E402
from paper_1808_08645_b200 import ElasticSolver, Solver2D  # noqa: E402
from workloads import elastic as ew  # noqa: E402
from workloads import kuhn, tri2d  # noqa: E402


def run2d(N, M, n, T=0.5):
    v, e = tri2d.tri_mesh(n)
    f = tri2d.c2_smooth_2d(1.0)
    c2 = tri2d.project_c2(v, e, f, M)
    s = Solver2D(v, e, N, M, c2)
    s.set_source(tri2d.manufactured_source(v, e, N, f))
    s.set_state(tri2d.manufactured_initial(v, e, N))
    dt0 = 0.5 * tri2d.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
    nst = int(np.ceil(T / dt0))
    s.run(0.0, T / nst, nst)
    err = Acoustic2DOracle(v, e, N, M, c2).l2_error(s.get_state(), tri2d.manufactured_exact, T)
    s.close()
    return err, len(e)


def run_el(N, M, n, T=0.25):
    v, e = kuhn.kuhn_mesh(n)
    mats = ew.constant_material(len(e), M, 1.0, 0.0, 0.5)
    s = ElasticSolver(v, e, N, M, *mats)
    s.set_state(ew.standing_p_wave_initial(v, e, N))
    dt0 = 0.5 * kuhn.min_height(v, e) / (N + 1) ** 2
    nst = int(np.ceil(T / dt0))
    s.run(0.0, T / nst, nst)
    o = ElasticOracle(v, e, N, M, *mats)
    Q = s.get_state()
    err = float(np.sqrt(sum(o.l2_error(Q, ew.standing_p_wave_exact, T, field=c) ** 2 for c in range(6))))
    s.close()
    return err, len(e)


out = {"two_d": [], "elastic": []}
for N in (4, 5):
    for M in (0, 1, 2, 3):
        errs, Ks = [], []
        for n in (4, 8, 16, 32):
            er, K = run2d(N, M, n)
            errs.append(er)
            Ks.append(K)
        rates = [float(np.log2(errs[i] / errs[i + 1])) for i in range(len(errs) - 1)]
        out["two_d"].append({"N": N, "M": M, "K": Ks, "L2_error": errs, "rates": rates,
                             "predicted": 2 if M == 0 else min(N + 1, M + 3)})
        print("2D", N, M, errs, rates, flush=True)
for N in (2, 3, 4, 5):
    errs, Ks = [], []
    for n in (2, 4, 8):
        er, K = run_el(N, 1, n)
        errs.append(er)
        Ks.append(K)
    rates = [float(np.log2(errs[i] / errs[i + 1])) for i in range(len(errs) - 1)]
    out["elastic"].append({"N": N, "M": 1, "K": Ks, "L2_error": errs, "rates": rates, "predicted": N + 1})
    print("elastic", N, errs, rates, flush=True)
json.dump(out, open(sys.argv[1], "w"), indent=1)
