"""Debug helper: per-element WADG/RHS parity of the CUDA path vs the oracle for a few (N, M)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '/root/repo')
from oracle.acoustic import AcousticOracle  # noqa: E402
from paper_1808_08645_b200 import Solver  # noqa: E402
from workloads import kuhn, media, states  # noqa: E402

cases = [tuple(int(x) for x in a.split(',')) for a in sys.argv[1:]] or [(4, 3)]
v, e = kuhn.kuhn_mesh(3)
for N, M in cases:
    c2 = media.random_c2(len(e), M)
    r = np.random.default_rng(7).standard_normal((len(e), states.num_coeffs(N)))
    o = AcousticOracle(v, e, N, M, c2)
    s = Solver(v, e, N, M, c2)
    out = s.wadg_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    ref = o.wadg(r)
    err = np.abs(out - ref).max(1)
    bad = np.nonzero(err > 1e-12)[0]
    print(N, M, 'bad elems', len(bad), bad[:10], 'max err', err.max(), flush=True)
