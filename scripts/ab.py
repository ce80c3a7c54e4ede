#!/usr/bin/env python
"""A/B tuning variants of libbbwadg.so (library vs library; no oracle).

    [AB_DTYPE=f32] [AB_NCUBE=n] python scripts/ab.py N M ref_variant var1 [var2 ...]

For every variant (a directory under paper_1808_08645_b200/native/, or `default`), a
subprocess computes one RHS and 3 LSRK steps on a random state of an n=6 Kuhn mesh and
times config-5-shaped stages; outputs are compared against `ref_variant` (relative L2).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, json, numpy as np, torch
sys.path.insert(0, ROOT)
from workloads.kuhn import kuhn_mesh
from workloads.media import random_c2
from workloads.states import random_state
from paper_1808_08645_b200.solver import Solver
N, M, tag, ncube = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
import os
dt = os.environ.get("AB_DTYPE", "f64")
v, e = kuhn_mesh(6)
s = Solver(v, e, N, M, random_c2(len(e), M), dtype=dt)
Q = torch.tensor(random_state(len(e), N), device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32)
r = s.rhs(Q).cpu().numpy()
s.set_state(random_state(len(e), N)); s.run(0.0, 1e-3, 3); q3 = s.get_state()
np.save(f"/tmp/ab_{tag}_rhs.npy", r); np.save(f"/tmp/ab_{tag}_q3.npy", np.asarray(q3))
s.close()
v, e = kuhn_mesh(ncube)
from workloads.media import project_c2, c2_smooth
s = Solver(v, e, N, M, random_c2(len(e), M, lo=0.9, hi=1.1), dtype=dt)
s.set_state(np.zeros((len(e), 4, (N+1)*(N+2)*(N+3)//6)))
s.run(0.0, 1e-4, 2); s.synchronize()
st = torch.cuda.Event(enable_timing=True); en = torch.cuda.Event(enable_timing=True)
best = 1e30
for rep in range(3):
    torch.cuda.synchronize(); st.record(); s.run(0.0, 1e-4, 2); en.record(); torch.cuda.synchronize()
    best = min(best, st.elapsed_time(en) / 10)
Np = (N+1)*(N+2)*(N+3)//6
print(json.dumps({"tag": tag, "ms_per_stage": best, "dofstage_per_s": 4*len(e)*Np/(best*1e-3)}))
'''


def main():
    N, M, ref = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    variants = [ref] + sys.argv[4:]
    ncube = int(os.environ.get("AB_NCUBE", "64"))
    import numpy as np
    res = {}
    for rep in range(int(os.environ.get("AB_REPS", "2"))):
        for vname in variants:
            lib = os.path.join(ROOT, "paper_1808_08645_b200", "native", "" if vname == "default" else vname, "libbbwadg.so")
            env = dict(os.environ, BBWADG_LIB=lib)
            out = subprocess.run([sys.executable, "-c", "ROOT=%r\n" % ROOT + CHILD, str(N), str(M), vname, str(ncube)],
                                 env=env, capture_output=True, text=True)
            if out.returncode != 0:
                print(vname, "FAILED", out.stderr[-2000:])
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res.setdefault(vname, []).append(d["dofstage_per_s"])
    r0 = np.load(f"/tmp/ab_{ref}_rhs.npy"); q0 = np.load(f"/tmp/ab_{ref}_q3.npy")
    for vname in variants:
        if vname not in res:
            continue
        r = np.load(f"/tmp/ab_{vname}_rhs.npy"); q = np.load(f"/tmp/ab_{vname}_q3.npy")
        er = np.linalg.norm(r - r0) / np.linalg.norm(r0); eq = np.linalg.norm(q - q0) / np.linalg.norm(q0)
        print(f"{vname:>12s} N={N} M={M}  {max(res[vname]):.3e} DOF-stage/s (reps {['%.3e' % x for x in res[vname]]})"
              f"  rhs rel {er:.1e}  3-step rel {eq:.1e}")


if __name__ == "__main__":
    main()
