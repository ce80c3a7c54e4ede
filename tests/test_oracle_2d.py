"""Pins of the 2D (triangle) oracle, oracle/acoustic2d.py, each against something
other than itself: closed forms and quadrature for the reference operators, finite differences for the
derivative, exact rational weighted projections, linear-field exactness of the RHS, the energy-rate identity
with independently evaluated edge jumps, and the paper's 2D convergence rates (r = 2 for M = 0,
min(N+1, M+3) for M >= 1) on its 2D manufactured solution."""
from fractions import Fraction
from math import comb

import numpy as np
import pytest

from oracle import acoustic2d as a2
from oracle import quadrature as qd
from workloads import tri2d

RNG = np.random.default_rng(20182)


@pytest.mark.parametrize("N", [1, 3, 6])
def test_mass_closed_form_equals_quadrature(N):
    lam, w = qd.tri_rule(N + 1)
    V = a2.eval_basis(N, lam)
    Mq = (V.T * (w * 2)) @ V
    assert np.max(np.abs(Mq.astype(np.float64) - a2.mass(N))) < 1e-15


@pytest.mark.parametrize("N", [1, 2, 5])
def test_derivative_matches_finite_differences(N):
    D = a2.derivative_ops(N)
    c = RNG.standard_normal(a2.num_coeffs(N))
    rs = np.array([[-0.5, -0.2], [0.1, -0.6], [-0.9, 0.5]])
    h = 1e-6
    def val(p):
        r, s = p[:, 0], p[:, 1]
        lam = np.stack([-(r + s) / 2, (1 + r) / 2, (1 + s) / 2], axis=1)
        return a2.eval_basis(N, lam) @ c
    for d in range(2):
        e = np.zeros(2)
        e[d] = h
        fd = (val(rs + e) - val(rs - e)) / (2 * h)
        r, s = rs[:, 0], rs[:, 1]
        lam = np.stack([-(r + s) / 2, (1 + r) / 2, (1 + s) / 2], axis=1)
        assert np.max(np.abs(a2.eval_basis(N, lam) @ (D[d] @ c) - fd)) < 1e-6


def _linear(X, N, a, b):
    idx = np.array(a2.multi_indices(N), dtype=float) / N
    pts = np.einsum("av,kvd->kad", idx, X)
    return pts @ a + b


@pytest.mark.parametrize("N", [1, 3])
def test_linear_velocity_gives_divergence(N):
    v, e = tri2d.tri_mesh(3)
    A, b = RNG.standard_normal((2, 2)), RNG.standard_normal(2)
    c2 = np.full((len(e), 3), 1.7)  # constant c^2 (M = 1 coefficients)
    o = a2.Acoustic2DOracle(v, e, N, 1, c2, tau_p=0.6, tau_u=1.4)
    Q = np.zeros((len(e), 3, a2.num_coeffs(N)))
    for c in range(2):
        Q[:, 1 + c] = _linear(o.mesh.X, N, A[c], b[c])
    R = o.rhs(Q)
    assert np.max(np.abs(R[:, 1:])) < 1e-12
    assert np.max(np.abs(R[:, 0] + 1.7 * np.trace(A))) < 1e-12


def test_linear_pressure_interior_elements():
    N = 3
    v, e = tri2d.tri_mesh(4)
    a = RNG.standard_normal(2)
    o = a2.Acoustic2DOracle(v, e, N, 1, np.ones((len(e), 3)))
    Q = np.zeros((len(e), 3, a2.num_coeffs(N)))
    Q[:, 0] = _linear(o.mesh.X, N, a, 0.3)
    R = o.rhs(Q)
    interior = np.all(o.mesh.nbr >= 0, axis=1)
    assert interior.sum() > 0
    assert np.max(np.abs(R[interior, 0])) < 1e-12
    for c in range(2):
        assert np.max(np.abs(R[interior, 1 + c] + a[c])) < 1e-12


def test_wadg_constant_weight_is_scaling():
    v, e = tri2d.tri_mesh(2)
    o = a2.Acoustic2DOracle(v, e, 4, 2, np.full((len(e), 6), 0.8))
    r = RNG.standard_normal((len(e), a2.num_coeffs(4)))
    assert np.max(np.abs(o.wadg(r) - 0.8 * r)) < 1e-13


@pytest.mark.parametrize("N,M", [(1, 1), (2, 1), (3, 2)])
def test_wadg_equals_exact_weighted_projection(N, M):
    # M^-1 M_{c^2} in rationals: int B^M_g B^N_a B^N_b = |T| C(a+b,a) C(a+b+g,g) / (C(2N,N) C(2N+M,M) C(2N+M+2,2))
    I, Im = a2.multi_indices(N), a2.multi_indices(M)
    c = [Fraction(int(x), 7) for x in RNG.integers(3, 12, size=len(Im))]
    s = Fraction(2, comb(2 * N, N) * comb(2 * N + M, M) * comb(2 * N + M + 2, 2))
    cab = lambda a, b: np.prod([comb(x + y, x) for x, y in zip(a, b)])  # noqa: E731
    Mc = [[sum(cg * int(cab(a, b)) * int(cab(tuple(x + y for x, y in zip(a, b)), g)) for cg, g in zip(c, Im)) * s
           for b in I] for a in I]
    Minv = a2.mass_inv_exact(N)
    W = [[sum(Minv[i][l] * Mc[l][j] for l in range(len(I))) for j in range(len(I))] for i in range(len(I))]
    v, e = tri2d.tri_mesh(1)
    o = a2.Acoustic2DOracle(v, e, N, M, np.array([[float(x) for x in c]] * len(e)))
    r = RNG.standard_normal((1, len(I)))
    want = r @ np.array([[float(x) for x in row] for row in W]).T
    assert np.max(np.abs(o.wadg(np.repeat(r, len(e), 0))[0] - want[0])) < 1e-13


def _edge_loss(v, e, N, Q, tau_p, tau_u):
    """-dE/dt from the edge jumps (Eq. sdf): interior edges int tau_p/2 [[p]]^2 + tau_u/2 [[u.n]]^2, boundary
    edges tau_p int p^2; own Gauss-Legendre points and affine maps."""
    X = v[e]
    t, w = np.polynomial.legendre.leggauss(N + 2)
    t, w = (t + 1) / 2, w / 2
    keys = {}
    for k in range(len(e)):
        for f in range(3):
            keys.setdefault(tuple(sorted((int(e[k][(f + 1) % 3]), int(e[k][(f + 2) % 3])))), []).append((k, f))

    def evaluate(k, x):
        E = np.stack([X[k, 1] - X[k, 0], X[k, 2] - X[k, 0]], axis=1)
        l = np.linalg.solve(E, (x - X[k, 0]).T).T
        lam = np.concatenate([1 - l.sum(1, keepdims=True), l], axis=1)
        return np.einsum("qi,ci->cq", a2.eval_basis(N, lam), Q[k])

    loss = 0.0
    for pairs in keys.values():
        k, f = pairs[0]
        A, B = X[k, (f + 1) % 3], X[k, (f + 2) % 3]
        x = A[None, :] * (1 - t)[:, None] + B[None, :] * t[:, None]
        L = np.linalg.norm(B - A)
        n = np.array([B[1] - A[1], -(B[0] - A[0])]) / L
        if np.dot(n, A - X[k, f]) < 0:
            n = -n
        qm = evaluate(k, x)
        if len(pairs) == 1:
            loss += tau_p * L * np.sum(w * qm[0] ** 2)
        else:
            qp = evaluate(pairs[1][0], x)
            jp, jun = qp[0] - qm[0], n @ (qp[1:3] - qm[1:3])
            loss += L * np.sum(w * (0.5 * tau_p * jp ** 2 + 0.5 * tau_u * jun ** 2))
    return loss


@pytest.mark.parametrize("tau", [(1.0, 1.0), (0.3, 2.0), (0.0, 0.0)])
def test_energy_rate_equals_penalty_edge_integrals(tau):
    N, M = 3, 1
    v, e = tri2d.tri_mesh(3)
    o = a2.Acoustic2DOracle(v, e, N, M, tri2d.random_c2(len(e), M), tau_p=tau[0], tau_u=tau[1])
    Q = np.random.default_rng(31).standard_normal((len(e), 3, a2.num_coeffs(N)))
    pred = -_edge_loss(v, e, N, Q, *tau)
    assert abs(o.energy_rate(Q) - pred) <= 1e-12 * max(abs(pred), o.energy(Q))


def test_energy_rate_pin_detects_doubled_penalty():
    N, M = 2, 1
    v, e = tri2d.tri_mesh(3)
    c2 = tri2d.random_c2(len(e), M)
    Q = np.random.default_rng(32).standard_normal((len(e), 3, a2.num_coeffs(N)))
    pred = -_edge_loss(v, e, N, Q, 1.0, 1.0)
    for tp, tu in [(2.0, 1.0), (1.0, 2.0)]:
        o = a2.Acoustic2DOracle(v, e, N, M, c2, tau_p=tp, tau_u=tu)
        assert abs(o.energy_rate(Q) - pred) > 1e-3 * abs(pred)


@pytest.mark.parametrize("N,M,rate", [(2, 1, 2.7), (2, 0, 1.8), (3, 1, 3.3)])
def test_manufactured_convergence_rate_2d(N, M, rate):
    # r = 2 (M = 0), min(N+1, M+3) (M >= 1), on the 2D manufactured solution P:646-652
    errs = []
    for n in (4, 8):
        v, e = tri2d.tri_mesh(n)
        f = tri2d.c2_smooth_2d(1.0)
        c2 = tri2d.project_c2(v, e, f, M)
        o = a2.Acoustic2DOracle(v, e, N, M, c2, source=tri2d.manufactured_source(v, e, N, f))
        T = 0.5
        dt0 = 0.5 * tri2d.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
        nst = int(np.ceil(T / dt0))
        Q = o.run(tri2d.manufactured_initial(v, e, N), 0.0, T / nst, nst)
        errs.append(o.l2_error(Q, tri2d.manufactured_exact, T))
    assert np.log2(errs[0] / errs[1]) > rate, errs
