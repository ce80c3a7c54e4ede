import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle.acoustic import AcousticOracle
from workloads import kuhn, media, states
from paper_1808_08645_b200 import Solver
v, e = kuhn.kuhn_mesh(2)
for N, M in [(1,0),(1,1),(2,0),(2,1),(3,0),(3,1),(5,0),(5,3),(7,0),(7,4)]:
    c2 = media.random_c2(len(e), M)
    r = np.random.default_rng(7).standard_normal((len(e), states.num_coeffs(N)))
    o = AcousticOracle(v, e, N, M, c2); s = Solver(v, e, N, M, c2)
    out = s.wadg_apply(torch.from_numpy(r).cuda()).cpu().numpy(); ref = o.wadg(r)
    Q = states.random_state(len(e), N)
    rr = s.rhs(torch.from_numpy(Q).cuda()).cpu().numpy(); rref = o.rhs(Q)
    print(N, M, 'wadg', np.linalg.norm(out-ref)/np.linalg.norm(ref), 'rhs', np.linalg.norm(rr-rref)/np.linalg.norm(rref))
    if np.linalg.norm(out-ref)/np.linalg.norm(ref) > 1e-10:
        print('  out0', np.round(out[0],4)); print('  ref0', np.round(ref[0],4))
