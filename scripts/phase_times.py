"""Per-phase cycle breakdown of the stage kernel (needs the BBW_PHASE_TIMING library variant).
   BBWADG_PHASE_TIMING=1 BBWADG_LIB=.../native/ptime/libbbwadg.so python scripts/phase_times.py N M n_cubes"""
import ctypes, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1808_08645_b200 import Solver, lib as L
from workloads import kuhn, media
N, M, n = (int(x) for x in sys.argv[1:4])
v, e = kuhn.kuhn_mesh(n)
c2 = media.project_c2(v, e, media.c2_smooth(1.0), M, device=torch.device("cuda"))
s = Solver(v, e, N, M, c2)
s.set_state(torch.randn((len(e), 4, (N+1)*(N+2)*(N+3)//6), dtype=torch.float64, device="cuda"))
f = L._L.bbwadg_debug_phase_times; f.restype = ctypes.c_int; f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
out = np.zeros(32, dtype=np.uint64)
s.step(0, 1e-4); f(s.ctx, out.ctypes.data)
for i in range(3): s.step(0, 1e-4)
f(s.ctx, out.ctypes.data)
names = ["A load", "B flux+grad", "C1/C2", "C3 L0", "D layers", "E gather+LSRKu", "F multiply", "G reductions", "H down", "I up", "J out"]
tot = out[:11].sum()
print(f"N={N} M={M} K={len(e)}: cycles per group-batch by phase (3 steps)")
for i, nm in enumerate(names):
    print(f"  {nm:16s} {out[i] / tot * 100:6.1f}%")
