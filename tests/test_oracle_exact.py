"""Exact-rational mini-oracle for BASELINE config 1: the whole right-hand side of
Eq. WADGform in Python Fractions, against the fp64 oracle (oracle/acoustic.py).

Independent of the oracle's construction: no quadrature, no numerical solve.  It uses
* the sparse barycentric derivative (d/d lambda_j of sum q_a B^N_a = N sum_b q_{b+e_j} B^{N-1}_b) and
  the degree elevation B^{N-1}_b = sum_j (b_j+1)/N B^N_{b+e_j} (Eq. bbele), where the oracle uses
  D = M^-1 S from a refined dense solve;
* closed-form simplex moments: int_T B^n_a B^m_b = |T| C(a+b,a) / (C(n+m,n) C(n+m+d,d)) and the Bernstein
  product rule for M_{c^2}, where the oracle uses quadrature;
* face traces as 2-D Bernstein polynomials (the trace on face f keeps the coefficients with a_f = 0,
  P:261), matched to the neighbour by GLOBAL vertex ids, where the oracle evaluates the neighbour's
  polynomial at physical quadrature points;
* an exact rational inverse of the reference mass matrix.
The penalties are 0 (central flux, Eq. sdf P:98-107 with tau = 0): every quantity is then rational on the
Kuhn mesh (area-weighted normals |f| n = cross / 2; the face-area factors cancel), so the result is exact;
the tau terms are pinned separately (energy-rate identity, tests/test_oracle_pins.py).
"""
from fractions import Fraction as Fr
from math import comb

import numpy as np

from oracle.acoustic import AcousticOracle
from workloads import kuhn, media, states


def idx3(n):  # canonical order (R19): a3, a2, a1 loops, a0 = n - a1 - a2 - a3
    return [(n - a1 - a2 - a3, a1, a2, a3) for a3 in range(n + 1) for a2 in range(n + 1 - a3)
            for a1 in range(n + 1 - a3 - a2)]


def mchoose(a, b):  # C(a+b, a) for multi-indices
    r = 1
    for x, y in zip(a, b):
        r *= comb(x + y, x)
    return r


def simplex_moment(n, m, d):  # int_T B^n_a B^m_b / |T| = C(a+b,a) / (C(n+m,n) C(n+m+d,d)) without C(a+b,a)
    return Fr(1, comb(n + m, n) * comb(n + m + d, d))


def mat_inv(A):
    n = len(A)
    M = [list(row) + [Fr(int(i == j)) for j in range(n)] for i, row in enumerate(A)]
    for c in range(n):
        p = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        piv = M[c][c]
        M[c] = [x / piv for x in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [x - f * y for x, y in zip(M[r], M[c])]
    return [row[n:] for row in M]


def matvec(A, x):
    return [sum((a * b for a, b in zip(row, x)), Fr(0)) for row in A]


def exact_rhs(v, e, N, M, c2, Q):
    """dQ/dt of Eq. WADGform with tau_p = tau_u = 0, in Fractions, for every element."""
    I_N, I_M, I_Nm1 = idx3(N), idx3(M), idx3(N - 1)
    pos = {a: i for i, a in enumerate(I_N)}
    posm1 = {a: i for i, a in enumerate(I_Nm1)}
    Np = len(I_N)
    # reference mass / |T| and its exact inverse
    mom = simplex_moment(N, N, 3)
    Mhat = [[mchoose(a, b) * mom for b in I_N] for a in I_N]
    Minv = mat_inv(Mhat)
    tri_mom = simplex_moment(N, N, 2)
    trip = Fr(1, comb(2 * N, N)) * simplex_moment(2 * N, M, 3)  # product rule + moment for int B^M B^N B^N
    V = [[Fr(x) for x in row] for row in np.asarray(v)]
    K = len(e)
    E = [[int(x) for x in row] for row in np.asarray(e)]
    # global face -> (element, face)
    faces = {}
    for k in range(K):
        for f in range(4):
            faces.setdefault(tuple(sorted(E[k][j] for j in range(4) if j != f)), []).append((k, f))
    Qf = [[[Fr(x) for x in Q[k, c]] for c in range(4)] for k in range(K)]

    def geometry(k):
        X = [V[E[k][i]] for i in range(4)]
        A = [[X[i + 1][d] - X[0][d] for i in range(3)] for d in range(3)]  # x = X0 + A l
        Ainv = mat_inv(A)  # l = Ainv (x - X0)
        grads = [[-sum(Ainv[i][d] for i in range(3)) for d in range(3)]] + [[Ainv[i][d] for d in range(3)] for i in range(3)]
        det = (A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0])
               + A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]))
        vol = det / 6
        return X, grads, vol

    def dphys(q, grads, x):
        """d/dx_x of the degree-N polynomial q (coefficients), as degree-N coefficients (P:264 + Eq. bbele)."""
        g = [Fr(0)] * len(I_Nm1)
        for ib, b in enumerate(I_Nm1):
            for j in range(4):
                bj = list(b)
                bj[j] += 1
                g[ib] += grads[j][x] * N * q[pos[tuple(bj)]]
        out = [Fr(0)] * Np
        for ib, b in enumerate(I_Nm1):
            for j in range(4):
                a = list(b)
                a[j] += 1
                out[pos[tuple(a)]] += Fr(b[j] + 1, N) * g[ib]
        return out

    def face_trace(k, f, q):
        """2-D Bernstein coefficients of the trace on face f, keyed by exponents on the face's GLOBAL vertex ids."""
        others = [j for j in range(4) if j != f]
        out = {}
        for a in I_N:
            if a[f] == 0:
                out[tuple(sorted((E[k][j], a[j]) for j in others))] = q[pos[a]]
        return out

    res = np.zeros(Q.shape)
    for k in range(K):
        X, grads, vol = geometry(k)
        p, u = Qf[k][0], Qf[k][1:4]
        rp = [Fr(0)] * Np
        for c in range(3):
            dc = dphys(u[c], grads, c)
            rp = [x - y for x, y in zip(rp, dc)]
        ru = [[-x for x in dphys(p, grads, c)] for c in range(3)]
        for f in range(4):
            others = [j for j in range(4) if j != f]
            P0, P1, P2 = (X[j] for j in others)
            e1 = [P1[d] - P0[d] for d in range(3)]
            e2 = [P2[d] - P0[d] for d in range(3)]
            cr = [e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]]
            if sum(cr[d] * (P0[d] - X[f][d]) for d in range(3)) < 0:
                cr = [-x for x in cr]
            an = [x / 2 for x in cr]  # |f| n (outward)
            key = tuple(sorted(E[k][j] for j in others))
            nbrs = [kf for kf in faces[key] if kf[0] != k]
            tm = [face_trace(k, f, q) for q in Qf[k]]
            if nbrs:
                kn, fn = nbrs[0]
                tp = [face_trace(kn, fn, q) for q in Qf[kn]]
            else:  # pressure release (R11): p+ = -p, u+ = u
                tp = [{kk: -x for kk, x in tm[0].items()}] + tm[1:]
            # |f| F_p = -1/2 (|f| n).[[u]],  |f| F_u = -1/2 |f| [[p]]; only the |f| F_u n_i = -1/2 (|f| n_i) [[p]] enters
            Fp = {kk: -Fr(1, 2) * sum(an[c] * (tp[1 + c][kk] - tm[1 + c][kk]) for c in range(3)) for kk in tm[0]}
            Fu_n = [{kk: -Fr(1, 2) * an[c] * (tp[0][kk] - tm[0][kk]) for kk in tm[0]} for c in range(3)]
            # int_f F phi_a / |f| for a with a_f = 0: 2-D moments in the face's vertex exponents
            def lift(F):
                rhs = [Fr(0)] * Np
                for a in I_N:
                    if a[f] != 0:
                        continue
                    ka = tuple(sorted((E[k][j], a[j]) for j in others))
                    ea = [x[1] for x in ka]
                    for kb, Fb in F.items():
                        eb = [x[1] for x in kb]
                        rhs[pos[a]] += Fb * mchoose(ea, eb) * tri_mom
                return [x / vol for x in matvec(Minv, rhs)]  # (M^k)^-1 = (|T| Mhat)^-1
            lp = lift(Fp)
            rp = [x + y for x, y in zip(rp, lp)]
            for c in range(3):
                lu = lift(Fu_n[c])
                ru[c] = [x + y for x, y in zip(ru[c], lu)]
        # WADG: (M^k)^-1 M^k_{c^2} = Mhat^-1 T_c, T_c[a][b] = sum_g c_g C(a+b,a) C(a+b+g,g) trip
        cg = [Fr(x) for x in c2[k]]
        Tc = [[sum((cg[ig] * mchoose(a, b) * mchoose(tuple(x + y for x, y in zip(a, b)), g) for ig, g in enumerate(I_M)),
                   Fr(0)) * trip for b in I_N] for a in I_N]
        dp = matvec(Minv, matvec(Tc, rp))
        res[k, 0] = [float(x) for x in dp]
        for c in range(3):
            res[k, 1 + c] = [float(x) for x in ru[c]]
    return res


def test_exact_rational_rhs_config1():
    # BASELINE config 1 mesh and degrees (48 tets, N = 3, M = 1), random state and c^2 coefficients
    # (fp64 values, taken exactly as rationals by both sides)
    v, e = kuhn.kuhn_mesh(2)
    N, M = 3, 1
    c2 = media.random_c2(len(e), M)
    Q = states.random_state(len(e), N)
    ref = exact_rhs(v, e, N, M, c2, Q)
    got = AcousticOracle(v, e, N, M, c2, tau_p=0.0, tau_u=0.0).rhs(Q)
    scale = np.max(np.abs(ref))
    assert np.max(np.abs(got - ref)) <= 1e-13 * scale, np.max(np.abs(got - ref)) / scale
    # per field, per element
    for c in range(4):
        assert np.max(np.abs(got[:, c] - ref[:, c])) <= 1e-13 * np.max(np.abs(ref[:, c]))


def test_exact_rational_rhs_n3_mesh_m2():
    # a 162-tet mesh with interior elements, N = 2, M = 2
    v, e = kuhn.kuhn_mesh(3)
    N, M = 2, 2
    c2 = media.random_c2(len(e), M)
    Q = states.random_state(len(e), N)
    ref = exact_rhs(v, e, N, M, c2, Q)
    got = AcousticOracle(v, e, N, M, c2, tau_p=0.0, tau_u=0.0).rhs(Q)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
