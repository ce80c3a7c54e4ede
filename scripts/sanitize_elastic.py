#!/usr/bin/env python
"""Small elastic BBWADG runs for compute-sanitizer: one RHS, one matrix-weighted WADG apply and two LSRK
steps at (N, M) on an n^3 Kuhn mesh.   python scripts/sanitize_elastic.py N M n [f64|f32]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_08645_b200 import ElasticSolver  # noqa: E402
from workloads import elastic as ew  # noqa: E402
from workloads import kuhn  # noqa: E402

N, M, n = (int(x) for x in sys.argv[1:4])
dt = sys.argv[4] if len(sys.argv) > 4 else "f64"
v, e = kuhn.kuhn_mesh(n)
mats = ew.random_material(len(e), M)
s = ElasticSolver(v, e, N, M, *mats, dtype=dt)
td = torch.float64 if dt == "f64" else torch.float32
Q = torch.tensor(ew.random_state(len(e), N), dtype=td, device="cuda")
r = s.rhs(Q)
w = s.wadg_apply(Q)
s.set_state(ew.random_state(len(e), N))
s.run(0.0, 1e-3, 2)
torch.cuda.synchronize()
print("ok", N, M, len(e), float(r.abs().max()), float(w.abs().max()), float(np.abs(s.get_state()).max()))
