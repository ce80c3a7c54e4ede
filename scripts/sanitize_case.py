#!/usr/bin/env python
"""Small BBWADG runs for compute-sanitizer (racecheck / synccheck / memcheck): one RHS, one WADG apply and
two LSRK steps at (N, M) on an n^3 Kuhn mesh.   python scripts/sanitize_case.py N M n [f64|f32]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_08645_b200 import Solver  # noqa: E402
from workloads import kuhn, media, states  # noqa: E402

N, M, n = (int(x) for x in sys.argv[1:4])
dt = sys.argv[4] if len(sys.argv) > 4 else "f64"
v, e = kuhn.kuhn_mesh(n)
c2 = media.random_c2(len(e), M)
s = Solver(v, e, N, M, c2, dtype=dt)
td = torch.float64 if dt == "f64" else torch.float32
Q = torch.tensor(states.random_state(len(e), N), dtype=td, device="cuda")
r = s.rhs(Q)
w = s.wadg_apply(Q[:, 0].contiguous())
s.set_state(states.random_state(len(e), N))
s.run(0.0, 1e-3, 2)
torch.cuda.synchronize()
print("ok", N, M, len(e), float(r.abs().max()), float(w.abs().max()), float(np.abs(s.get_state()).max()))
