"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every oracle function is checked here against something other than itself
(closed forms, exact rational arithmetic, complex-step derivatives, invariants,
special cases that reduce to textbook results).  A plausible mistake anywhere
in the oracle -- a dropped term, a wrong sign or index, a transposed operand --
fails at least one test.  DESIGN.md "Oracle pins" maps each test to the
oracle function and the paper passage.
"""
from fractions import Fraction
from math import comb

import numpy as np
import pytest

from oracle import bernstein as bb
from oracle import operators as ops
from oracle import quadrature as qd
from oracle.acoustic import AcousticOracle, lsrk_stability_polynomial
from workloads import kuhn, media, states

RNG = np.random.default_rng(20180823)


# --------------------------------------------------------------------------- basis
@pytest.mark.parametrize("N", [1, 2, 4, 7])
def test_partition_of_unity_and_nonnegativity(N):
    # P:69 "forms a nonnegative partition of unity"
    lam = RNG.dirichlet([1, 1, 1, 1], size=100)
    B = bb.eval_basis(N, lam)
    assert np.all(B >= 0)
    assert np.max(np.abs(B.sum(1) - 1)) < 1e-14


def test_vertex_property_and_count():
    B = bb.eval_basis(1, np.eye(4))
    assert np.array_equal(B, np.eye(4))  # B^1_{e_j}(vertex i) = delta_ij
    for n in range(10):
        assert len(bb.multi_indices(n)) == comb(n + 3, 3)
        assert all(sum(a) == n and min(a) >= 0 for a in bb.multi_indices(n))


def test_product_of_basis_functions():
    # B^N_a B^M_b = C(a+b, a)/C(N+M, N) B^{N+M}_{a+b}
    lam = RNG.dirichlet([1, 1, 1, 1], size=30)
    for N, M in [(1, 1), (2, 1), (3, 2)]:
        BN, BM, BNM = bb.eval_basis(N, lam), bb.eval_basis(M, lam), bb.eval_basis(N + M, lam)
        idx = {a: i for i, a in enumerate(bb.multi_indices(N + M))}
        for i, a in enumerate(bb.multi_indices(N)):
            for j, b in enumerate(bb.multi_indices(M)):
                g = tuple(x + y for x, y in zip(a, b))
                coef = Fraction(np.prod([comb(g[k], a[k]) for k in range(4)]), comb(N + M, N))
                assert np.allclose(BN[:, i] * BM[:, j], float(coef) * BNM[:, idx[g]], rtol=1e-14, atol=0)
    # the tiny cases of P:300: B^1_ei B^1_ej = 1/2 B^2_{ei+ej} (i != j), (B^1_ei)^2 = B^2_{2ei}
    B1, B2 = bb.eval_basis(1, lam), bb.eval_basis(2, lam)
    i2 = {a: i for i, a in enumerate(bb.multi_indices(2))}
    e = np.eye(4, dtype=int)
    for i in range(4):
        for j in range(4):
            g = tuple(e[i] + e[j])
            assert np.allclose(B1[:, i] * B1[:, j], (1.0 if i == j else 0.5) * B2[:, i2[g]], rtol=1e-15)


def test_mass_matrix_closed_form_matches_moment_formula_and_quadrature():
    # M_ij = int phi_i phi_j: integer form == Fraction moments == 40-digit quadrature
    for n in [1, 2, 3]:
        A, s = bb.mass_integer(n)
        Mex = bb.mass_exact(n)
        for i in range(A.shape[0]):
            for j in range(A.shape[1]):
                assert s * int(A[i, j]) == Mex[i][j]
        lam, w = qd.tet_rule(n + 1)
        V = bb.eval_basis(n, lam)
        Mq = (V.T * w) @ V * np.longdouble(4) / 3
        Mf = np.array([[float(x) for x in r] for r in Mex])
        assert np.max(np.abs(Mq.astype(float) - Mf)) < 1e-16 * np.max(Mf) * 10


# --------------------------------------------------------------------------- quadrature
@pytest.mark.parametrize("q", [1, 3, 6])
def test_tet_rule_exact_to_2q_minus_1(q):
    lam, w = qd.tet_rule(q)
    deg = 2 * q - 1
    for a in bb.multi_indices(deg):  # every degree-(2q-1) barycentric monomial (homogeneous => all lower too)
        approx = float(np.sum(w * np.prod(lam ** np.array(a, dtype=np.longdouble), axis=1)))
        exact = float(bb.simplex_moment(a, 3))
        assert abs(approx - exact) < 1e-17 + 1e-15 * exact
    assert abs(float(w.sum()) - 1.0) < 1e-18


def test_tet_rule_not_exact_beyond():
    q = 3
    lam, w = qd.tet_rule(q)
    a = (0, 2 * q, 0, 0)
    approx = float(np.sum(w * lam[:, 1] ** (2 * q)))
    assert abs(approx - float(bb.simplex_moment(a))) > 1e-8


@pytest.mark.parametrize("q", [1, 4])
def test_triangle_rule_exact(q):
    lam, w = qd.tri_rule(q)
    deg = 2 * q - 1
    for a3 in range(deg + 1):
        for a2 in range(deg + 1 - a3):
            a = (deg - a2 - a3, a2, a3)
            approx = float(np.sum(w * np.prod(lam ** np.array(a, dtype=np.longdouble), axis=1)))
            assert abs(approx - float(bb.simplex_moment(a, 2))) < 1e-17


# --------------------------------------------------------------------------- operators
@pytest.mark.parametrize("N", [1, 3, 6])
def test_derivative_matrices_match_complex_step(N):
    # D_d = M^-1 S_d is exact differentiation on P^N: compare with the
    # complex-step derivative of the Bernstein expansion (independent of M, S)
    D = ops.derivative_ops(N)
    c = RNG.standard_normal(bb.num_coeffs(N))
    rst = RNG.dirichlet([1, 1, 1, 1], size=40)[:, 1:] * 2 - 1
    h = 1e-30
    for d in range(3):
        z = rst.astype(complex)
        z[:, d] += 1j * h
        dv = (bb.eval_basis(N, bb.barycentric_from_ref(z)) @ c).imag / h
        num = bb.eval_basis(N, bb.barycentric_from_ref(rst)) @ (D[d] @ c)
        assert np.max(np.abs(num - dv)) < 1e-14 * np.max(np.abs(dv))


def test_derivative_sparsity_bound():
    # each row of a barycentric derivative has <= d+1 nonzeros; D_r = (D^1 - D^0)/2
    # therefore has <= 2(d+1) - shared nonzeros; at least it must be far from dense
    for N in [3, 5]:
        D = ops.derivative_ops(N)
        nnz = (np.abs(D) > 1e-10).sum(axis=2)
        assert nnz.max() <= 8


@pytest.mark.parametrize("N", [2, 4])
def test_lift_is_M_inverse_face_mass(N):
    # L^f = M^-1 M_f: M L'_f (V_f g) = |T^| * (int_f g phi_j / |f^|), exact rational face moments
    lams, Vf, Lf = ops.face_ops(N)
    Mh = ops.mass(N)
    idx = bb.multi_indices(N)
    g = RNG.standard_normal(len(idx))
    for f in range(4):
        lhs = Mh @ (Lf[f] @ (Vf[f] @ g))
        rhs = np.zeros(len(idx))
        for j, a in enumerate(idx):
            if a[f] != 0:
                continue
            for i, b in enumerate(idx):
                if b[f] != 0:
                    continue
                ab = [x + y for k, (x, y) in enumerate(zip(a, b)) if k != f]
                mom = bb.simplex_moment(ab, 2)  # normalised face measure
                rhs[j] += float(bb.REF_VOLUME * bb.multinomial(a) * bb.multinomial(b) * mom) * g[i]
        assert np.max(np.abs(lhs - rhs)) < 1e-13 * np.max(np.abs(rhs))


def _triple_exact(N, M):
    """T[c][a][b] = int B^M_c B^N_a B^N_b (exact Fractions, moment formula)."""
    iN, iM = bb.multi_indices(N), bb.multi_indices(M)
    T = np.empty((len(iM), len(iN), len(iN)), dtype=object)
    for c, g in enumerate(iM):
        for i, a in enumerate(iN):
            for j, b in enumerate(iN):
                e = tuple(x + y + z for x, y, z in zip(a, b, g))
                T[c, i, j] = bb.REF_VOLUME * bb.multinomial(a) * bb.multinomial(b) * bb.multinomial(g) * bb.simplex_moment(e)
    return T


@pytest.mark.parametrize("N,M", [(1, 1), (2, 1), (3, 1), (2, 2)])
def test_wadg_equals_exact_weighted_projection(N, M):
    # Eq. pwadg with an exact rule == M^-1 M_{c^2} computed in exact rationals
    import sympy

    v, e = kuhn.kuhn_mesh(1)
    c2 = media.random_c2(len(e), M)
    o = AcousticOracle(v, e, N, M, c2)
    T = _triple_exact(N, M)
    Mex = sympy.Matrix(bb.mass_exact(N))
    Minv = Mex.inv()
    r = RNG.standard_normal((len(e), bb.num_coeffs(N)))
    got = o.wadg(r)
    for k in range(2):
        cf = [Fraction(x) for x in c2[k]]
        Mc = sympy.Matrix([[sum(cf[c] * T[c, i, j] for c in range(T.shape[0])) for j in range(T.shape[2])]
                           for i in range(T.shape[1])])
        W = np.array((Minv * Mc).evalf(30), dtype=float)
        assert np.max(np.abs(got[k] - W @ r[k])) < 1e-14 * np.max(np.abs(W @ r[k]))


def test_wadg_constant_weight_is_scaling():
    # constant c^2 -> (M^k_{1/c^2})^-1 M^k = c^2 I (standard DG)
    v, e = kuhn.kuhn_mesh(1)
    for N, M in [(3, 1), (5, 3), (7, 4)]:
        kappa = 1.7
        c2 = np.full((len(e), bb.num_coeffs(M)), kappa)  # constant in Bernstein = all coeffs equal
        o = AcousticOracle(v, e, N, M, c2)
        r = RNG.standard_normal((len(e), bb.num_coeffs(N)))
        assert np.max(np.abs(o.wadg(r) - kappa * r)) < 2e-13 * np.max(np.abs(r))


def test_wadg_operator_is_M_selfadjoint_positive():
    # M W = M_{c^2} is symmetric positive definite for positive c^2
    v, e = kuhn.kuhn_mesh(1)
    N, M = 4, 2
    o = AcousticOracle(v, e, N, M, media.random_c2(len(e), M))
    Mh = ops.mass(N)
    for k in range(3):
        oo = AcousticOracle(v, e[k:k + 1], N, M, o.c2M[k:k + 1])
        Wk = np.stack([oo.wadg(col[None])[0] for col in np.eye(bb.num_coeffs(N))], axis=1)
        S = Mh @ Wk
        assert np.max(np.abs(S - S.T)) < 1e-12 * np.max(np.abs(S))
        assert np.min(np.linalg.eigvalsh(0.5 * (S + S.T))) > 0


# --------------------------------------------------------------------------- right-hand side
def _linear_field_coeffs(X, N, a, b):
    """Bernstein coefficients of the global linear field a.x + b on every element:
    the value at the domain point sum_v (alpha_v/N) X_v (exact for linear fields)."""
    idx = bb.index_array(N).astype(float) / N
    pts = np.einsum("av,kvd->kad", idx, X)
    return pts @ a + b


@pytest.mark.parametrize("N", [1, 3])
def test_rhs_linear_velocity_gives_divergence(N):
    # p = 0, u = A x + b (global, continuous): all jumps vanish (also on the pressure-release
    # boundary, u+ = u, p+ = -p = 0), so dp/dt = -c^2-weighted div u and du/dt = 0 exactly.
    v, e = kuhn.kuhn_mesh(2)
    A = RNG.standard_normal((3, 3))
    b = RNG.standard_normal(3)
    M = 1
    c2 = np.ones((len(e), bb.num_coeffs(M)))
    o = AcousticOracle(v, e, N, M, c2, tau_p=0.7, tau_u=1.3)
    X = o.mesh.X
    Q = np.zeros((len(e), 4, bb.num_coeffs(N)))
    for c in range(3):
        Q[:, 1 + c] = _linear_field_coeffs(X, N, A[c], b[c])
    R = o.rhs(Q)
    assert np.max(np.abs(R[:, 1:])) < 1e-12
    assert np.max(np.abs(R[:, 0] + np.trace(A))) < 1e-12


def test_rhs_linear_pressure_interior_elements():
    # p = a.x + b, u = 0: interior faces have no jumps, so on elements without boundary
    # faces du/dt = -grad p = -a and dp/dt = 0 exactly.
    N, M = 3, 1
    v, e = kuhn.kuhn_mesh(3)
    a = RNG.standard_normal(3)
    o = AcousticOracle(v, e, N, M, np.ones((len(e), 4)))
    Q = np.zeros((len(e), 4, bb.num_coeffs(N)))
    Q[:, 0] = _linear_field_coeffs(o.mesh.X, N, a, 0.3)
    R = o.rhs(Q)
    interior = np.all(o.mesh.nbr >= 0, axis=1)
    assert interior.sum() > 0
    assert np.max(np.abs(R[interior, 0])) < 1e-12
    for c in range(3):
        assert np.max(np.abs(R[interior, 1 + c] + a[c])) < 1e-12


@pytest.mark.parametrize("N,M", [(2, 1), (3, 2)])
def test_energy_conservation_central_flux(N, M):
    # tau = 0 with p+ = -p, u+ = u: the semi-discrete scheme is energy conservative
    # (skew-symmetric in the WADG energy norm; R22)
    v, e = kuhn.kuhn_mesh(2)
    o = AcousticOracle(v, e, N, M, media.random_c2(len(e), M), tau_p=0.0, tau_u=0.0)
    for s in range(3):
        Q = np.random.default_rng(s).standard_normal((len(e), 4, bb.num_coeffs(N)))
        assert abs(o.energy_rate(Q)) < 1e-12 * o.energy(Q)


@pytest.mark.parametrize("tau", [(1.0, 1.0), (0.5, 2.0)])
def test_energy_dissipation_upwind(tau):
    # tau >= 0 makes the scheme dissipative; dE/dt = -sum_f int tau_p/2 [[p]]^2 + tau_u/2 [[u.n]]^2 (per face pair)
    N, M = 3, 1
    v, e = kuhn.kuhn_mesh(2)
    o = AcousticOracle(v, e, N, M, media.random_c2(len(e), M), tau_p=tau[0], tau_u=tau[1])
    for s in range(3):
        Q = np.random.default_rng(s).standard_normal((len(e), 4, bb.num_coeffs(N)))
        assert o.energy_rate(Q) < 0


def test_energy_non_increasing_in_time():
    N, M = 3, 1
    v, e = kuhn.kuhn_mesh(2)
    o = AcousticOracle(v, e, N, M, media.random_c2(len(e), M))
    Q = states.random_state(len(e), N)
    res = np.zeros_like(Q)
    dt = 0.5 * kuhn.min_height(v, e) / (np.sqrt(1.5) * (N + 1) ** 2)
    E0 = o.energy(Q)
    for it in range(5):
        o.step(Q, res, it * dt, dt)
        E1 = o.energy(Q)
        assert E1 <= E0 * (1 + 1e-14)
        E0 = E1


# --------------------------------------------------------------------------- time integrator
def test_lsrk_stability_polynomial():
    # order 4 on linear problems: R(z) = 1 + z + z^2/2 + z^3/6 + z^4/24 + O(z^5) ("4th order")
    R = lsrk_stability_polynomial()
    exact = [1, 1, Fraction(1, 2), Fraction(1, 6), Fraction(1, 24)]
    assert len(R) == 6
    for k in range(5):
        assert abs(float(R[k] - exact[k])) < 1e-12
    assert abs(float(R[5]) - 1 / 200) < 1e-10  # Carpenter-Kennedy (5,4): z^5 coefficient 1/200


# --------------------------------------------------------------------------- convergence
@pytest.mark.slow
def test_manufactured_convergence_rate():
    # rate r = min(N+1, M+3) for M >= 1.  N=2, M=2 -> 3 (2.26, 2.99 pre-asymptotic)
    N, M = 2, 2
    errs = []
    for n in [4, 8]:
        v, e = kuhn.kuhn_mesh(n)
        f = media.c2_smooth(1.0)
        c2 = media.project_c2(v, e, f, M)
        g = states.manufactured_source(v, e, N, f)
        o = AcousticOracle(v, e, N, M, c2, source=g)
        Q0 = states.manufactured_initial(v, e, N)
        T = 0.5
        dt0 = 0.5 * kuhn.min_height(v, e) / (np.sqrt(c2.max()) * (N + 1) ** 2)
        nst = int(np.ceil(T / dt0))
        Q = o.run(Q0, 0.0, T / nst, nst)
        errs.append(o.l2_error(Q, states.manufactured_exact, T))
    rate = np.log2(errs[0] / errs[1])
    assert rate > 2.7, (errs, rate)


# --------------------------------------------------------------------------- penalty scale (Eq. sdf)
def _face_energy_loss(v, e, N, Q, tau_p, tau_u):
    """-dE/dt predicted from the face jumps alone (Eq. sdf; derivation in DESIGN.md §3):
    summing p r_p + u.r_u over the two sides of an interior face, the central parts cancel and
    -int_f (tau_p/2 [[p]]^2 + tau_u/2 [[u.n]]^2) remains; on a pressure-release boundary face
    (p+ = -p, u+ = u, R11) the sum is -tau_p int_f p^2.  Computed here from physical face points,
    the test's own affine maps and normals (no oracle operator is used)."""
    X = v[e]  # K,4,3
    K = len(e)
    keys = {}
    for k in range(K):
        for f in range(4):
            keys.setdefault(tuple(sorted(int(x) for j, x in enumerate(e[k]) if j != f)), []).append((k, f))
    lam3, w = qd.tri_rule(N + 1)  # exact to degree 2N+1 on the face
    lam3 = lam3.astype(np.float64)
    w = w.astype(np.float64)

    def evaluate(k, x):  # fields of element k at physical points x[nq,3]
        E = np.stack([X[k, 1] - X[k, 0], X[k, 2] - X[k, 0], X[k, 3] - X[k, 0]], axis=1)
        l = np.linalg.solve(E, (x - X[k, 0]).T).T
        lam = np.concatenate([1 - l.sum(1, keepdims=True), l], axis=1)
        return np.einsum("qi,ci->cq", bb.eval_basis(N, lam), Q[k])

    loss = 0.0
    for pairs in keys.values():
        k, f = pairs[0]
        others = [j for j in range(4) if j != f]
        P3 = X[k, others]
        x = lam3 @ P3
        cr = np.cross(P3[1] - P3[0], P3[2] - P3[0])
        area = 0.5 * np.linalg.norm(cr)
        n = cr / np.linalg.norm(cr)
        if np.dot(n, P3[0] - X[k, f]) < 0:
            n = -n
        qm = evaluate(k, x)
        if len(pairs) == 1:
            loss += tau_p * area * np.sum(w * qm[0] ** 2)
        else:
            qp = evaluate(pairs[1][0], x)
            jp = qp[0] - qm[0]
            jun = n @ (qp[1:4] - qm[1:4])
            loss += area * np.sum(w * (0.5 * tau_p * jp ** 2 + 0.5 * tau_u * jun ** 2))
    return loss


@pytest.mark.parametrize("tau", [(1.0, 1.0), (0.5, 2.0), (0.0, 3.0)])
def test_energy_rate_equals_penalty_face_integrals(tau):
    # pins the penalty SCALE of Eq. sdf, not only its sign: dE/dt = -sum of the face
    # integrals of tau_p/2 [[p]]^2 + tau_u/2 [[u.n]]^2 (interior) and tau_p p^2 (boundary)
    N, M = 3, 1
    v, e = kuhn.kuhn_mesh(2)
    o = AcousticOracle(v, e, N, M, media.random_c2(len(e), M), tau_p=tau[0], tau_u=tau[1])
    for s in range(2):
        Q = np.random.default_rng(100 + s).standard_normal((len(e), 4, bb.num_coeffs(N)))
        pred = -_face_energy_loss(v, e, N, Q, *tau)
        assert abs(o.energy_rate(Q) - pred) <= 1e-12 * abs(pred), (o.energy_rate(Q), pred)


def test_energy_rate_pin_detects_penalty_mutation():
    # mutation check of the pin above: an oracle whose penalty is doubled (the "dropped 1/2" class
    # of mistakes on tau) must fail it
    N, M = 2, 1
    v, e = kuhn.kuhn_mesh(2)
    c2 = media.random_c2(len(e), M)
    Q = np.random.default_rng(7).standard_normal((len(e), 4, bb.num_coeffs(N)))
    pred = -_face_energy_loss(v, e, N, Q, 1.0, 1.0)
    for tp, tu in [(2.0, 1.0), (1.0, 2.0)]:
        o = AcousticOracle(v, e, N, M, c2, tau_p=tp, tau_u=tu)
        assert abs(o.energy_rate(Q) - pred) > 1e-3 * abs(pred)


# --------------------------------------------------------------------------- LSRK stage times
def _lsrk_scalar(A, B, C, f, t0, dt):
    """One 2N-storage step of y' = f(t) (y-independent), exact rational arithmetic."""
    y, res = Fraction(0), Fraction(0)
    for s in range(5):
        res = A[s] * res + dt * f(t0 + C[s] * dt)
        y = y + B[s] * res
    return y


def test_lsrk_stage_times_are_the_implied_abscissae():
    # c_s is the time the stage input represents: the stage-s value of y' = 1, y(0) = 0, dt = 1
    # (P:1264 cites Carpenter-Kennedy; R13)
    from oracle.acoustic import LSRK_A, LSRK_B, LSRK_C
    y, res = Fraction(0), Fraction(0)
    for s in range(5):
        assert abs(float(y - LSRK_C[s])) < 1e-11, (s, float(y), float(LSRK_C[s]))
        res = LSRK_A[s] * res + 1
        y = y + LSRK_B[s] * res
    assert abs(float(y) - 1.0) < 1e-11


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_lsrk_integrates_polynomials_in_time(k):
    # 4th order: y' = k t^(k-1) is integrated exactly for k <= 4 -- this uses the stage
    # times, which the stability polynomial cannot see
    from oracle.acoustic import LSRK_A, LSRK_B, LSRK_C
    y = _lsrk_scalar(LSRK_A, LSRK_B, LSRK_C, lambda t: k * t ** (k - 1), Fraction(0), Fraction(1))
    assert abs(float(y) - 1.0) < 1e-11
    # mutation check: c_3 * (1 + 1e-6) breaks it for k >= 2
    if k >= 2:
        C = list(LSRK_C)
        C[3] = C[3] * (1 + Fraction(1, 10 ** 6))
        y = _lsrk_scalar(LSRK_A, LSRK_B, C, lambda t: k * t ** (k - 1), Fraction(0), Fraction(1))
        assert abs(float(y) - 1.0) > 1e-8


def test_oracle_step_uses_stage_times():
    # a time-dependent source makes the stage times visible: the oracle's step must equal the
    # 2N-storage recursion evaluated at t0 + c_s dt with c_s the abscissae IMPLIED by (A, B)
    # (computed here, not read from LSRK_C)
    from oracle.acoustic import LSRK_A, LSRK_B
    N, M = 2, 1
    v, e = kuhn.kuhn_mesh(2)
    c2 = media.random_c2(len(e), M)
    g = np.random.default_rng(3).standard_normal((len(e), bb.num_coeffs(N)))
    o = AcousticOracle(v, e, N, M, c2, source=g)
    c, y, r = [], Fraction(0), Fraction(0)
    for s in range(5):
        c.append(float(y))
        r = LSRK_A[s] * r + 1
        y = y + LSRK_B[s] * r
    t0, dt = 0.3, 0.05
    Q0 = 1e-3 * np.random.default_rng(4).standard_normal((len(e), 4, bb.num_coeffs(N)))
    Q = o.run(Q0, t0, dt, 1)
    q, res = Q0.copy(), np.zeros_like(Q0)
    for s in range(5):
        res = float(LSRK_A[s]) * res + dt * o.rhs(q, t0 + c[s] * dt)
        q = q + float(LSRK_B[s]) * res
    assert np.max(np.abs(Q - q)) <= 1e-13 * np.max(np.abs(q))
    # the source term is not negligible here: shifting c_3 by 1e-6 moves the result above that bar
    res, q2 = np.zeros_like(Q0), Q0.copy()
    for s in range(5):
        cs = c[s] * (1 + 1e-6) if s == 3 else c[s]
        res = float(LSRK_A[s]) * res + dt * o.rhs(q2, t0 + cs * dt)
        q2 = q2 + float(LSRK_B[s]) * res
    assert np.max(np.abs(q2 - q)) > 1e-12 * np.max(np.abs(q))


# --------------------------------------------------------------------------- diagnostics
def test_energy_with_constant_wavespeed_is_plain_l2():
    # R22 / P:136-137: for constant c^2 the WADG norm p^T M M_{c^2}^-1 M p reduces to int p^2 / c^2, so
    # E = 1/2 sum_k [int p^2 / c^2 + int |u|^2], computed here by an independent quadrature (workloads'
    # Stroud rule, exact to 2N+7) of the evaluated fields
    from workloads.errors import l2_error

    N, M, cval = 3, 0, 1.7
    v, e = kuhn.kuhn_mesh(2)
    c2 = np.full((len(e), 1), cval)
    o = AcousticOracle(v, e, N, M, c2)
    Q = np.random.default_rng(5).standard_normal((len(e), 4, bb.num_coeffs(N)))
    zero = lambda x, y, z: 0.0 * x  # noqa: E731
    ip = l2_error(v, e, Q[:, 0], N, zero) ** 2
    iu = sum(l2_error(v, e, Q[:, c], N, zero) ** 2 for c in (1, 2, 3))
    ref = 0.5 * (ip / cval + iu)
    assert abs(o.energy(Q) - ref) <= 1e-12 * ref


def test_oracle_l2_error_matches_independent_quadrature():
    # the oracle's error norm (R18) against workloads.errors (its own rule and basis evaluation)
    from workloads.errors import l2_error

    N = 3
    v, e = kuhn.kuhn_mesh(2)
    o = AcousticOracle(v, e, N, 1, media.random_c2(len(e), 1))
    Q = np.random.default_rng(6).standard_normal((len(e), 4, bb.num_coeffs(N)))
    f = lambda x, y, z, t: (np.sin(x + 2 * y) * np.cos(z - t), 0, 0, 0)  # noqa: E731
    a = o.l2_error(Q, f, 0.3, q=N + 6)
    b = l2_error(v, e, Q[:, 0], N, lambda x, y, z: f(x, y, z, 0.3)[0], q=N + 6)
    assert abs(a - b) <= 1e-12 * b
