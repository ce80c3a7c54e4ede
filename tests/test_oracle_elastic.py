"""Pins of the elastic CPU oracle (oracle/elastic.py).

Each part of the elastic right-hand side is checked against something other than itself:
* volume terms sum_i A_i^T d_i sigma and sum_i A_i d_i v: exact on globally linear fields, against the
  closed-form strain / divergence written out here (a transposed A_i or a dropped term fails);
* the matrix-weighted WADG update (I x M^-1) M_C: equals C r for constant Lame parameters (P:134
  analogue) and equals the sum of the PINNED scalar acoustic WADG operators over the blocks C_st;
* the whole scheme: with mu = 0, rho = 1, lambda = c^2, tau_v = 0 it reduces to the pinned acoustic
  oracle (p = -s11 = -s22 = -s33, u = v), Eq. ewave -> Eq. awave;
* the penalty fluxes: the semi-discrete energy rate equals minus the face integrals of
  tau_v/2 |A_n [[v]]|^2 + tau_s/2 |A_n^T [[sigma]]|^2 (interior) and tau_s |A_n^T sigma|^2 (traction-free
  boundary), computed here from physical face points; zero with tau = 0; doubled penalties fail it;
* the time-discrete solution converges at rate ~N+1 to the exact standing P-wave (R27).
"""
import numpy as np
import pytest

from oracle import bernstein as bb
from oracle import quadrature as qd
from oracle.acoustic import AcousticOracle
from oracle.elastic import A_MATS, ElasticOracle, isotropic_C
from workloads import elastic as ew
from workloads import kuhn, media

RNG = np.random.default_rng(20180824)


def _linear_field_coeffs(X, N, a, b):
    # Bernstein coefficients of a linear function = its values at the equispaced lattice points (exact)
    idx = bb.index_array(N).astype(float) / N
    pts = np.einsum("av,kvd->kad", idx, X)
    return pts @ a + b


def _voigt_strain(G):
    """(e11, e22, e33, 2 e23, 2 e13, 2 e12) of the velocity gradient G[a, i] = d v_a / d x_i."""
    return np.array([G[0, 0], G[1, 1], G[2, 2], G[1, 2] + G[2, 1], G[0, 2] + G[2, 0], G[0, 1] + G[1, 0]])


@pytest.mark.parametrize("N", [1, 3])
def test_linear_velocity_gives_stress_rate_C_strain(N):
    # v = G x + b continuous, sigma = 0: no jumps anywhere (v+ = v, sigma+ = -0 on the boundary), so
    # dv/dt = 0 and dsigma/dt = C eps(v) exactly on every element (Hooke's law of Eq. ewave)
    v, e = kuhn.kuhn_mesh(2)
    M = 1
    lam, mu = 0.8, 0.35
    mats = ew.constant_material(len(e), M, 1.3, lam, mu)
    o = ElasticOracle(v, e, N, M, *mats, tau_v=0.6, tau_s=1.7)
    G = RNG.standard_normal((3, 3))
    b = RNG.standard_normal(3)
    Q = np.zeros((len(e), 9, bb.num_coeffs(N)))
    for a in range(3):
        Q[:, a] = _linear_field_coeffs(o.mesh.X, N, G[a], b[a])
    R = o.rhs(Q)
    assert np.max(np.abs(R[:, 0:3])) < 1e-12
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[np.arange(3), np.arange(3)] += 2 * mu
    C[np.arange(3, 6), np.arange(3, 6)] = mu
    want = C @ _voigt_strain(G)
    for s in range(6):
        assert np.max(np.abs(R[:, 3 + s] - want[s])) < 1e-12


def test_linear_stress_gives_divergence_on_interior_elements():
    # sigma = linear, v = 0: interior faces have no jumps, so there rho dv/dt = div sigma exactly:
    # (d1 s11 + d2 s12 + d3 s13, d1 s12 + d2 s22 + d3 s23, d1 s13 + d2 s23 + d3 s33)
    N, M = 3, 1
    v, e = kuhn.kuhn_mesh(3)
    rho_inv = 0.7
    o = ElasticOracle(v, e, N, M, *ew.constant_material(len(e), M, rho_inv, 1.0, 0.5))
    S = RNG.standard_normal((6, 3))  # d sigma_s / d x_i
    Q = np.zeros((len(e), 9, bb.num_coeffs(N)))
    for s in range(6):
        Q[:, 3 + s] = _linear_field_coeffs(o.mesh.X, N, S[s], 0.1 * s)
    R = o.rhs(Q)
    interior = np.all(o.mesh.nbr >= 0, axis=1)
    assert interior.sum() > 0
    # Voigt rows: 0 s11, 1 s22, 2 s33, 3 s23, 4 s13, 5 s12
    div = np.array([S[0, 0] + S[5, 1] + S[4, 2], S[5, 0] + S[1, 1] + S[3, 2], S[4, 0] + S[3, 1] + S[2, 2]])
    for a in range(3):
        assert np.max(np.abs(R[interior, a] - rho_inv * div[a])) < 1e-12
    assert np.max(np.abs(R[interior, 3:])) < 1e-12


def test_A_matrices_are_the_voigt_strain_operator():
    # sum_i A_i d_i v must be the engineering strain: check on a random gradient
    G = RNG.standard_normal((3, 3))
    assert np.allclose(np.einsum("isa,ai->s", A_MATS, G), _voigt_strain(G), atol=1e-15)


def test_constant_material_wadg_is_C_times_r():
    N, M = 3, 2
    v, e = kuhn.kuhn_mesh(2)
    lam, mu, ri = 1.2, 0.4, 0.8
    o = ElasticOracle(v, e, N, M, *ew.constant_material(len(e), M, ri, lam, mu))
    r = RNG.standard_normal((len(e), 6, bb.num_coeffs(N)))
    C = isotropic_C(lam, mu)
    assert np.max(np.abs(o.wadg_sigma(r) - np.einsum("st,ktn->ksn", C, r))) < 1e-12
    assert np.max(np.abs(o.wadg_v(r[:, 0]) - ri * r[:, 0])) < 1e-12


@pytest.mark.parametrize("N,M", [(2, 1), (3, 2)])
def test_matrix_weighted_wadg_is_the_sum_of_scalar_wadg_blocks(N, M):
    # (I x M^-1) M_C r: block (s, t) is the scalar WADG operator with weight C_st, whose
    # degree-M coefficients are the same linear combination of the lambda, mu coefficients
    v, e = kuhn.kuhn_mesh(2)
    rho_inv, lam, mu = ew.random_material(len(e), M)
    o = ElasticOracle(v, e, N, M, rho_inv, lam, mu)
    r = RNG.standard_normal((len(e), 6, bb.num_coeffs(N)))
    Ccoef = isotropic_C(lam, mu)  # K, Mp, 6, 6: C is linear in (lambda, mu) coefficient-wise
    want = np.zeros_like(r)
    for s in range(6):
        for t in range(6):
            if np.all(Ccoef[:, :, s, t] == 0):
                continue
            ao = AcousticOracle(o.mesh, None, N, M, Ccoef[:, :, s, t])
            want[:, s] += ao.wadg(r[:, t])
    assert np.max(np.abs(o.wadg_sigma(r) - want)) < 1e-12 * np.max(np.abs(want))
    ao = AcousticOracle(o.mesh, None, N, M, rho_inv)
    assert np.max(np.abs(o.wadg_v(r[:, 0]) - ao.wadg(r[:, 0]))) < 1e-12 * np.max(np.abs(r))


@pytest.mark.parametrize("N,M,tau", [(2, 1, 1.0), (3, 2, 0.5)])
def test_mu_zero_reduces_to_acoustic(N, M, tau):
    # mu = 0, rho = 1, lambda = c^2: Eq. ewave with sigma = -p I is Eq. awave (u = v); the fluxes
    # reduce to Eq. sdf with tau_p = tau_s, tau_u = 0 (tau_v = 0), the WADG update to P_q c^2 V_q
    v, e = kuhn.kuhn_mesh(2)
    K = len(e)
    c2 = media.random_c2(K, M)
    mp = bb.num_coeffs(M)
    el = ElasticOracle(v, e, N, M, np.ones((K, mp)), c2, np.zeros((K, mp)), tau_v=0.0, tau_s=tau)
    ac = AcousticOracle(el.mesh, None, N, M, c2, tau_p=tau, tau_u=0.0)
    Qa = np.random.default_rng(5).standard_normal((K, 4, bb.num_coeffs(N)))
    Qe = np.zeros((K, 9, bb.num_coeffs(N)))
    Qe[:, 0:3] = Qa[:, 1:4]
    Qe[:, 3:6] = -Qa[:, 0:1]
    Ra, Re = ac.rhs(Qa), el.rhs(Qe)
    scale = np.max(np.abs(Ra))
    assert np.max(np.abs(Re[:, 0:3] - Ra[:, 1:4])) < 1e-12 * scale
    for s in range(3):
        assert np.max(np.abs(Re[:, 3 + s] + Ra[:, 0])) < 1e-12 * scale
    assert np.max(np.abs(Re[:, 6:9])) < 1e-12 * scale


def _face_energy_loss(v, e, N, Q, tau_v, tau_s):
    """-dE/dt from the face jumps alone (derivation in DESIGN.md §3, elastic): on an interior face the
    central parts of the two sides cancel with the volume terms (integration by parts of
    v.A_i^T d_i sigma + sigma.A_i d_i v) and int tau_v/2 |A_n [[v]]|^2 + tau_s/2 |A_n^T [[sigma]]|^2
    remains; on a traction-free boundary face (sigma+ = -sigma, v+ = v) tau_s int |A_n^T sigma|^2.
    Physical face points, the test's own affine maps and normals (no oracle operator)."""
    X = v[e]
    K = len(e)
    keys = {}
    for k in range(K):
        for f in range(4):
            keys.setdefault(tuple(sorted(int(x) for j, x in enumerate(e[k]) if j != f)), []).append((k, f))
    lam3, w = qd.tri_rule(N + 1)
    lam3 = lam3.astype(np.float64)
    w = w.astype(np.float64)

    def evaluate(k, x):
        E = np.stack([X[k, 1] - X[k, 0], X[k, 2] - X[k, 0], X[k, 3] - X[k, 0]], axis=1)
        l = np.linalg.solve(E, (x - X[k, 0]).T).T
        lam = np.concatenate([1 - l.sum(1, keepdims=True), l], axis=1)
        return np.einsum("qi,ci->cq", bb.eval_basis(N, lam), Q[k])

    def An(n):  # A_n = sum_i n_i A_i, written out from P:159-183
        return np.array([[n[0], 0, 0], [0, n[1], 0], [0, 0, n[2]], [0, n[2], n[1]], [n[2], 0, n[0]],
                         [n[1], n[0], 0]])

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
        A = An(n)
        qm = evaluate(k, x)
        if len(pairs) == 1:
            t = A.T @ qm[3:9]
            loss += tau_s * area * np.sum(w * np.sum(t * t, axis=0))
        else:
            qp = evaluate(pairs[1][0], x)
            jv = A @ (qp[0:3] - qm[0:3])
            jt = A.T @ (qp[3:9] - qm[3:9])
            loss += area * np.sum(w * (0.5 * tau_v * np.sum(jv * jv, 0) + 0.5 * tau_s * np.sum(jt * jt, 0)))
    return loss


@pytest.mark.parametrize("tau", [(1.0, 1.0), (0.5, 2.0), (0.0, 3.0), (2.5, 0.0)])
def test_energy_rate_equals_penalty_face_integrals(tau):
    N, M = 2, 1
    v, e = kuhn.kuhn_mesh(2)
    o = ElasticOracle(v, e, N, M, *ew.random_material(len(e), M), tau_v=tau[0], tau_s=tau[1])
    for s in range(2):
        Q = np.random.default_rng(200 + s).standard_normal((len(e), 9, bb.num_coeffs(N)))
        pred = -_face_energy_loss(v, e, N, Q, *tau)
        assert abs(o.energy_rate(Q) - pred) <= 1e-12 * abs(pred), (o.energy_rate(Q), pred)


def test_energy_rate_pin_detects_penalty_mutation():
    N, M = 2, 1
    v, e = kuhn.kuhn_mesh(2)
    mats = ew.random_material(len(e), M)
    Q = np.random.default_rng(9).standard_normal((len(e), 9, bb.num_coeffs(N)))
    pred = -_face_energy_loss(v, e, N, Q, 1.0, 1.0)
    for tv, ts in [(2.0, 1.0), (1.0, 2.0)]:
        o = ElasticOracle(v, e, N, M, *mats, tau_v=tv, tau_s=ts)
        assert abs(o.energy_rate(Q) - pred) > 1e-3 * abs(pred)


@pytest.mark.parametrize("N,M", [(2, 1), (3, 2)])
def test_energy_conservation_central_flux(N, M):
    # tau = 0: the scheme is skew-symmetric in the WADG energy norm (energy stable)
    v, e = kuhn.kuhn_mesh(2)
    o = ElasticOracle(v, e, N, M, *ew.random_material(len(e), M), tau_v=0.0, tau_s=0.0)
    for s in range(2):
        Q = np.random.default_rng(s).standard_normal((len(e), 9, bb.num_coeffs(N)))
        assert abs(o.energy_rate(Q)) < 1e-12 * o.energy(Q)


def test_energy_non_increasing_in_time():
    N, M = 2, 1
    v, e = kuhn.kuhn_mesh(2)
    mats = ew.random_material(len(e), M)
    o = ElasticOracle(v, e, N, M, *mats)
    Q = ew.random_state(len(e), N)
    res = np.zeros_like(Q)
    cp = np.sqrt((mats[1].max() + 2 * mats[2].max()) * mats[0].max())
    dt = 0.5 * kuhn.min_height(v, e) / (cp * (N + 1) ** 2)
    E0 = o.energy(Q)
    for it in range(4):
        o.step(Q, res, it * dt, dt)
        E1 = o.energy(Q)
        assert E1 <= E0 * (1 + 1e-14)
        E0 = E1


@pytest.mark.slow
def test_standing_p_wave_convergence_rate():
    # exact standing P-wave (R27: lambda = 0, mu = 1/2, rho = 1, traction-free box)
    N, M = 2, 1
    errs = []
    for n in [2, 4]:
        v, e = kuhn.kuhn_mesh(n)
        o = ElasticOracle(v, e, N, M, *ew.constant_material(len(e), M, 1.0, 0.0, 0.5))
        Q0 = ew.standing_p_wave_initial(v, e, N)
        T = 0.25
        dt0 = 0.5 * kuhn.min_height(v, e) / (1.0 * (N + 1) ** 2)
        nst = int(np.ceil(T / dt0))
        Q = o.run(Q0, 0.0, T / nst, nst)
        errs.append(np.sqrt(sum(o.l2_error(Q, ew.standing_p_wave_exact, T, field=c) ** 2 for c in range(6))))
    rate = np.log2(errs[0] / errs[1])
    assert rate > 2.6, (errs, rate)
