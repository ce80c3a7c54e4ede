"""BASELINE config 2 on the GPU path: O(h^{N+1}) convergence to the manufactured solution.

P:678: the L2 error converges at rate min(N+1, M+3) = N+1 for M = N.  The CUDA library runs every
step (source included, reading R17); the error is evaluated by workloads.errors (R18).  Rates are
checked between the n = 4 and n = 8 Kuhn meshes (384 -> 3072 tets) with a pre-asymptotic margin,
and the n = 8 error is compared with the CPU oracle's on the same mesh.
"""
import numpy as np
import pytest

from workloads import errors, kuhn, media, states

pytestmark = pytest.mark.gpu


def _gpu_error(N, n, T=0.5, M=None):
    from paper_1808_08645_b200 import Solver

    M = N if M is None else M
    v, e = kuhn.kuhn_mesh(n)
    f = media.c2_smooth(1.0)
    c2 = media.project_c2(v, e, f, M)
    s = Solver(v, e, N, M, c2)
    s.set_source(states.manufactured_source(v, e, N, f))
    s.set_state(states.manufactured_initial(v, e, N))
    dt0 = 0.5 * kuhn.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
    nst = int(np.ceil(T / dt0))
    s.run(0.0, T / nst, nst)
    Q = np.asarray(s.get_state())
    s.close()
    return errors.l2_error(v, e, Q[:, 0], N, lambda x, y, z: states.manufactured_exact(x, y, z, T)[0])


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_convergence_rate_N_plus_1(gpu_lib, N):
    e4, e8 = _gpu_error(N, 4), _gpu_error(N, 8)
    rate = np.log2(e4 / e8)
    assert rate > N + 1 - 0.6, (N, e4, e8, rate)


def test_gpu_error_equals_oracle_error(gpu_lib):
    # the same discrete solution: errors agree to far below the discretisation error
    from oracle.acoustic import AcousticOracle

    N = M = 2
    n, T = 4, 0.25
    v, e = kuhn.kuhn_mesh(n)
    f = media.c2_smooth(1.0)
    c2 = media.project_c2(v, e, f, M)
    g = states.manufactured_source(v, e, N, f)
    Q0 = states.manufactured_initial(v, e, N)
    dt0 = 0.5 * kuhn.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
    nst = int(np.ceil(T / dt0))
    o = AcousticOracle(v, e, N, M, c2, source=g)
    Qo = o.run(Q0, 0.0, T / nst, nst)
    from paper_1808_08645_b200 import Solver

    s = Solver(v, e, N, M, c2)
    s.set_source(g)
    s.set_state(Q0)
    s.run(0.0, T / nst, nst)
    Qg = np.asarray(s.get_state())
    s.close()
    ex = lambda x, y, z: states.manufactured_exact(x, y, z, T)[0]  # noqa: E731
    eo = errors.l2_error(v, e, Qo[:, 0], N, ex)
    eg = errors.l2_error(v, e, Qg[:, 0], N, ex)
    assert abs(eo - eg) <= 1e-9 * eo, (eo, eg)
    assert abs(eo - o.l2_error(Qo, states.manufactured_exact, T, q=N + 4)) <= 1e-12 * eo  # same rule, same norm


@pytest.mark.parametrize("N,M,rmin", [(4, 0, 1.6), (4, 1, 3.4), (5, 1, 3.4)])
def test_convergence_rate_M_below_N(gpu_lib, N, M, rmin):
    # r = 2 for M = 0 and min(N+1, M+3) for M >= 1 (M = 1: 4), between n = 8 and n = 16
    # (3,072 -> 24,576 tets; the paper's coarsest step is pre-asymptotic for M = 0 as well)
    e8, e16 = _gpu_error(N, 8, M=M), _gpu_error(N, 16, M=M)
    rate = np.log2(e8 / e16)
    predicted = 2 if M == 0 else min(N + 1, M + 3)
    assert rmin < rate < predicted + 0.8, (N, M, e8, e16, rate)
