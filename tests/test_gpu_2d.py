"""Parity of the 2D (triangle) CUDA path (bbwadg2d_setup + the common C ABI calls) against the pinned 2D oracle
(oracle/acoustic2d.py, tests/test_oracle_2d.py).

Tolerances as in 3D (BASELINE.json north_star): fp64 relative L2 <= 1e-12 per RHS / WADG apply, <= 1e-10
after steps, fp32 <= 1e-5; per-field, per-element maxima are asserted beside the pooled norm.
Inputs: random states (rng 2808), random c^2 Bernstein coefficients in [0.5, 1.5] (rng 2809), square meshes
of n x n x 2 triangles; n = 6 (72) and n = 40 (3,200 triangles: more than one wave of the persistent grid
for N >= 5, so its grid-stride loop iterates).
"""
import numpy as np
import pytest

from oracle.acoustic2d import Acoustic2DOracle
from workloads import tri2d

pytestmark = pytest.mark.gpu

CASES = sorted({(N, M) for N in range(1, 10) for M in (0, 1, N // 2 + 1, N) if M <= N})


def rel_l2(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def field_max_rel(a, b):
    return max(float(np.max(np.abs(a[:, c] - b[:, c])) / max(np.max(np.abs(b[:, c])), 1e-300))
               for c in range(b.shape[1]))


def _solver(v, e, N, M, c2, **kw):
    from paper_1808_08645_b200 import Solver2D

    return Solver2D(v, e, N, M, c2, **kw)


@pytest.fixture(scope="module")
def mesh6():
    return tri2d.tri_mesh(6)


@pytest.mark.parametrize("N,M", CASES)
def test_2d_rhs_parity(gpu_lib, mesh6, N, M):
    import torch

    v, e = mesh6
    c2 = tri2d.random_c2(len(e), M)
    Q = tri2d.random_state(len(e), N)
    o = Acoustic2DOracle(v, e, N, M, c2)
    s = _solver(v, e, N, M, c2)
    out = s.rhs(torch.from_numpy(Q).cuda(), 0.0).cpu().numpy()
    ref = o.rhs(Q)
    assert rel_l2(out, ref) <= 1e-12
    assert field_max_rel(out, ref) <= 1e-11


@pytest.mark.parametrize("N,M", [(1, 1), (3, 2), (5, 3), (7, 4), (9, 9), (4, 0)])
def test_2d_wadg_apply_parity(gpu_lib, mesh6, N, M):
    import torch

    v, e = mesh6
    c2 = tri2d.random_c2(len(e), M)
    r = np.random.default_rng(5).standard_normal((len(e), tri2d.num_coeffs(N)))
    o = Acoustic2DOracle(v, e, N, M, c2)
    out = _solver(v, e, N, M, c2).wadg_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert rel_l2(out, o.wadg(r)) <= 1e-12


@pytest.mark.parametrize("N,M,tau", [(2, 1, (0.0, 0.0)), (4, 2, (0.5, 2.0)), (7, 3, (2.0, 0.25))])
def test_2d_rhs_penalty_variants(gpu_lib, mesh6, N, M, tau):
    import torch

    v, e = mesh6
    c2 = tri2d.random_c2(len(e), M)
    Q = tri2d.random_state(len(e), N)
    o = Acoustic2DOracle(v, e, N, M, c2, tau_p=tau[0], tau_u=tau[1])
    out = _solver(v, e, N, M, c2, tau_p=tau[0], tau_u=tau[1]).rhs(torch.from_numpy(Q).cuda(), 0.0).cpu().numpy()
    assert rel_l2(out, o.rhs(Q)) <= 1e-12


def _dt(v, e, N, c2):
    return 0.5 * tri2d.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)


@pytest.mark.parametrize("N,M,n,steps", [(3, 1, 6, 20), (5, 3, 6, 10), (7, 4, 40, 2), (9, 9, 6, 3), (2, 2, 40, 3)])
def test_2d_steps_parity(gpu_lib, N, M, n, steps):
    v, e = tri2d.tri_mesh(n)
    c2 = tri2d.random_c2(len(e), M)
    Q0 = tri2d.random_state(len(e), N)
    dt = _dt(v, e, N, c2)
    o = Acoustic2DOracle(v, e, N, M, c2)
    s = _solver(v, e, N, M, c2)
    s.set_state(Q0)
    s.run(0.0, dt, steps)
    got, ref = s.get_state(), o.run(Q0, 0.0, dt, steps)
    assert rel_l2(got, ref) <= 1e-10
    assert field_max_rel(got, ref) <= 1e-9


@pytest.mark.parametrize("N,M", [(3, 1), (6, 3)])
def test_2d_fp32(gpu_lib, mesh6, N, M):
    import torch

    v, e = mesh6
    c2 = tri2d.random_c2(len(e), M)
    Q = tri2d.random_state(len(e), N)
    o = Acoustic2DOracle(v, e, N, M, c2)
    s = _solver(v, e, N, M, c2, dtype="f32")
    out = s.rhs(torch.from_numpy(Q.astype(np.float32)).cuda(), 0.0).cpu().numpy().astype(np.float64)
    assert rel_l2(out, o.rhs(Q)) <= 1e-5
    dt = _dt(v, e, N, c2)
    s.set_state(Q)
    s.run(0.0, dt, 3)
    assert rel_l2(s.get_state().astype(np.float64), o.run(Q, 0.0, dt, 3)) <= 1e-5


def test_2d_time_dependent_source(gpu_lib, mesh6):
    # manufactured source through bbwadg_set_source: stage times enter as sin(pi t_s)
    v, e = mesh6
    N, M = 4, 2
    f = tri2d.c2_smooth_2d(1.0)
    c2 = tri2d.project_c2(v, e, f, M)
    g = tri2d.manufactured_source(v, e, N, f)
    Q0 = tri2d.manufactured_initial(v, e, N)
    o = Acoustic2DOracle(v, e, N, M, c2, source=g)
    s = _solver(v, e, N, M, c2)
    s.set_source(g)
    s.set_state(Q0)
    dt = _dt(v, e, N, c2)
    s.run(0.1, dt, 5)
    assert rel_l2(s.get_state(), o.run(Q0, 0.1, dt, 5)) <= 1e-11


@pytest.mark.parametrize("N,M,rate", [(3, 1, 3.3), (4, 0, 1.8), (5, 2, 4.5)])
def test_2d_convergence_rates_on_gpu(gpu_lib, N, M, rate):
    # P:678 in 2D (Fig. con2d analogue on square meshes): r = 2 for M = 0, min(N+1, M+3) for M >= 1
    errs = []
    for n in (8, 16):
        v, e = tri2d.tri_mesh(n)
        f = tri2d.c2_smooth_2d(1.0)
        c2 = tri2d.project_c2(v, e, f, M)
        o = Acoustic2DOracle(v, e, N, M, c2)  # error norm only
        s = _solver(v, e, N, M, c2)
        s.set_source(tri2d.manufactured_source(v, e, N, f))
        s.set_state(tri2d.manufactured_initial(v, e, N))
        T = 0.5
        nst = int(np.ceil(T / _dt(v, e, N, c2)))
        s.run(0.0, T / nst, nst)
        errs.append(o.l2_error(s.get_state(), tri2d.manufactured_exact, T))
    assert np.log2(errs[0] / errs[1]) > rate, errs


def test_2d_energy_non_increasing_on_gpu(gpu_lib, mesh6):
    v, e = mesh6
    N, M = 4, 2
    c2 = tri2d.random_c2(len(e), M)
    o = Acoustic2DOracle(v, e, N, M, c2)
    s = _solver(v, e, N, M, c2)
    s.set_state(tri2d.random_state(len(e), N))
    dt = _dt(v, e, N, c2)
    E0 = o.energy(s.get_state())
    for _ in range(5):
        s.run(0.0, dt, 1)
        E1 = o.energy(s.get_state())
        assert E1 <= E0 * (1 + 1e-13)
        E0 = E1


def test_2d_setup_validates(gpu_lib, mesh6):
    from paper_1808_08645_b200 import lib as L

    v, e = mesh6
    c2 = tri2d.random_c2(len(e), 1)
    with pytest.raises(L.BBWADGError):  # clockwise triangles are rejected
        _solver(v, e[:, [0, 2, 1]], 3, 1, c2)
    with pytest.raises(L.BBWADGError):  # non-positive c^2
        _solver(v, e, 3, 1, -c2)
    with pytest.raises(ValueError):
        _solver(v, e, 3, 1, c2[:, :2])


def _closure2(e, sample):
    """sample triangles plus every triangle sharing an edge with one of them."""
    K = e.shape[0]
    edges = np.concatenate([np.sort(e[:, [1, 2]], 1), np.sort(e[:, [0, 2]], 1), np.sort(e[:, [0, 1]], 1)])
    owner = np.concatenate([np.arange(K)] * 3)
    order = np.lexsort((edges[:, 1], edges[:, 0]))
    se, so = edges[order], owner[order]
    same = np.all(se[1:] == se[:-1], axis=1)
    a, b = so[:-1][same], so[1:][same]
    want = np.zeros(K, dtype=bool)
    want[sample] = True
    return np.unique(np.concatenate([sample, b[want[a]], a[want[b]]]))


@pytest.mark.parametrize("N,M,dtype,tol", [(7, 4, "f64", 1e-12), (7, 4, "f32", 1e-5), (9, 2, "f64", 1e-12),
                                           (3, 1, "f64", 1e-12)])
def test_2d_full_size_sampled_parity(gpu_lib, N, M, dtype, tol):
    """bench.py's 2D workload at full size (n = 512, 524,288 triangles, smooth c^2) in the bench launch
    configuration: one bbwadg_rhs; the oracle recomputes 48 sampled triangles (with their edge neighbours)."""
    import torch

    n = 512
    v, e = tri2d.tri_mesh(n)
    c2 = tri2d.project_c2(v, e, tri2d.c2_smooth_2d(1.0), M)
    dev = torch.device("cuda", 0)
    s = _solver(v, e, N, M, c2, dtype=dtype)
    gen = torch.Generator(device=dev)
    gen.manual_seed(2808)
    Q = torch.randn((len(e), 3, tri2d.num_coeffs(N)), dtype=torch.float64, device=dev, generator=gen)
    if dtype == "f32":
        Q = Q.float()
    out = s.rhs(Q, 0.0)
    rng = np.random.default_rng(7)
    sample = np.unique(np.concatenate([rng.choice(len(e), 46, replace=False), [0, len(e) - 1]]))
    sub = _closure2(e, sample)
    idx = torch.from_numpy(sub).to(dev)
    Qs = Q.index_select(0, idx).double().cpu().numpy()
    got = out.index_select(0, idx).double().cpu().numpy()
    del out, Q
    s.close()
    ref = Acoustic2DOracle(v, e[sub], N, M, c2[sub]).rhs(Qs)
    pos = np.searchsorted(sub, sample)
    assert rel_l2(got[pos], ref[pos]) <= tol
    assert field_max_rel(got[pos], ref[pos]) <= 10 * tol
