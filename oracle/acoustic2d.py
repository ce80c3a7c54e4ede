"""Oracle WADG acoustic solver on TRIANGLES (2D) -- TEST INFRASTRUCTURE ONLY.

The 2D analogue of oracle/acoustic.py ("only one order of complexity can be reduced in two
dimensions"; 2D manufactured solution P:646-652, Fig. con2d).  Plain dense definitions, fp64 per
element, reference operators formed EXACTLY in rationals and rounded once:

* reference triangle D^ = {r, s >= -1, r + s <= 0}, vertices (-1,-1), (1,-1), (-1,1), |D^| = 2,
  l0 = -(r+s)/2, l1 = (1+r)/2, l2 = (1+s)/2;  B^N_a = N!/(a0! a1! a2!) l^a  (P:67-69 with d = 2);
  canonical order for a2: for a1: a0 = N - a1 - a2 (R29);
* mass M^ = |D^| C(a+b,a) / (C(2N,N) C(2N+2,2)) (closed-form simplex moments), stiffness
  S_d[i][j] = int B_i dB_j/dr_d from the same moments (dB^N_j = N sum_k dl_k B^{N-1}_{j-e_k}), D_d = M^-1 S_d
   -- exact Fractions, then fp64;
* lift L'_f = |D^| M^-1 V_f^T diag(w_f): (M^k)^-1 int_f F phi = (|f| / |T|) L'_f F(x_q) on a Gauss-Legendre
  edge rule; the neighbour's polynomial is evaluated at the SAME physical edge points through its inverse
  affine map (no orientation tables);
* WADG P_q diag(c^2_M(x_q)) V_q (Eq. pwadg, weight c^2: R1) on a collapsed rule exact to 2N+M
  (exactly the L2 projection of c^2_M r_p onto P^N that BBWADG computes);
* Eq. sdf fluxes, pressure-release boundary (R11), source placement R17, LSRK of oracle.acoustic.

Pins: tests/test_oracle_2d.py.
"""
from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache

import numpy as np
from mpmath import mp

from .acoustic import LSRK_A, LSRK_B, LSRK_C
from . import quadrature as qd

REF_AREA = Fraction(2)
# d(l_i)/d(r, s), i = 0, 1, 2
DL = ((Fraction(-1, 2), Fraction(-1, 2)), (Fraction(1, 2), Fraction(0)), (Fraction(0), Fraction(1, 2)))


def num_coeffs(n: int) -> int:
    return (n + 1) * (n + 2) // 2


@lru_cache(maxsize=None)
def multi_indices(n: int) -> tuple:
    return tuple((n - a1 - a2, a1, a2) for a2 in range(n + 1) for a1 in range(n + 1 - a2))


def _multinomial(a) -> int:
    return math.factorial(sum(a)) // math.prod(math.factorial(x) for x in a)


def eval_basis(n: int, lam: np.ndarray) -> np.ndarray:
    """B^n_a at barycentric points lam[..., 3] -> [..., Np2(n)] (dtype of lam)."""
    idx = np.array(multi_indices(n), dtype=np.int64)
    C = np.array([_multinomial(a) for a in multi_indices(n)], dtype=lam.dtype)
    return C * np.prod(lam[..., None, :] ** idx.astype(lam.dtype), axis=-1)


def _cab(a, b) -> int:
    return math.prod(math.comb(x + y, x) for x, y in zip(a, b))


def _frac_inv(A):
    n = len(A)
    M = [list(r) + [Fraction(int(i == j)) for j in range(n)] for i, r in enumerate(A)]
    for c in range(n):
        p = next(r for r in range(c, n) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        pv = M[c][c]
        M[c] = [x / pv for x in M[c]]
        for r in range(n):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [x - f * y for x, y in zip(M[r], M[c])]
    return [r[n:] for r in M]


@lru_cache(maxsize=None)
def mass_exact(n: int):
    """M^_{ab} = int_D^ B^n_a B^n_b (Fractions)."""
    I = multi_indices(n)
    s = REF_AREA / (math.comb(2 * n, n) * math.comb(2 * n + 2, 2))
    return tuple(tuple(s * _cab(a, b) for b in I) for a in I)


@lru_cache(maxsize=None)
def mass_inv_exact(n: int):
    return tuple(tuple(r) for r in _frac_inv([list(r) for r in mass_exact(n)]))


def mass(n: int) -> np.ndarray:
    return np.array([[float(x) for x in r] for r in mass_exact(n)])


@lru_cache(maxsize=None)
def derivative_ops(n: int) -> np.ndarray:
    """D_r, D_s = M^-1 S_d, exact then fp64, [2, Np2, Np2]."""
    I, Im = multi_indices(n), multi_indices(n - 1)
    s_mix = REF_AREA / (math.comb(2 * n - 1, n) * math.comb(2 * n + 1, 2))  # int B^n_a B^{n-1}_b / C(a+b,a)
    Minv = mass_inv_exact(n)
    out = []
    for d in range(2):
        S = [[Fraction(0)] * len(I) for _ in I]
        for j, b in enumerate(I):
            for k in range(3):
                if b[k] == 0 or DL[k][d] == 0:
                    continue
                bm = list(b)
                bm[k] -= 1
                for i, a in enumerate(I):
                    S[i][j] += n * DL[k][d] * _cab(a, bm) * s_mix
        D = [[sum((Minv[i][l] * S[l][j] for l in range(len(I))), Fraction(0)) for j in range(len(I))] for i in range(len(I))]
        out.append([[float(x) for x in r] for r in D])
    return np.array(out)


def _gauss01(q: int):
    with mp.workdps(40):
        X, W = mp.gauss_quadrature(q, "legendre")
        return ([np.longdouble(mp.nstr((x + 1) / 2, 30)) for x in X], [np.longdouble(mp.nstr(w / 2, 30)) for w in W])


@lru_cache(maxsize=None)
def edge_ops(n: int):
    """Per reference edge f (opposite vertex f): barycentric edge points [nq,3], V_f [nq, Np2], L'_f [Np2, nq]."""
    t, w = _gauss01(n + 1)  # exact to degree 2n+1 on the edge
    t, w = np.array(t, dtype=np.longdouble), np.array(w, dtype=np.longdouble)
    Minv = np.array([[np.longdouble(x.numerator) / np.longdouble(x.denominator) for x in r] for r in mass_inv_exact(n)])
    lams, Vs, Ls = [], [], []
    for f in range(3):
        a, b = (f + 1) % 3, (f + 2) % 3
        lam = np.zeros((len(t), 3), dtype=np.longdouble)
        lam[:, a] = 1 - t
        lam[:, b] = t
        V = eval_basis(n, lam)
        L = Minv @ (V.T * (w * np.longdouble(2))[None, :])
        lams.append(lam.astype(np.float64))
        Vs.append(V.astype(np.float64))
        Ls.append(L.astype(np.float64))
    return lams, Vs, Ls


@lru_cache(maxsize=None)
def wadg_ops(n: int, m: int):
    """V_q^n, V_q^m, P_q = M^-1 V_q^T diag(w |D^|) on the triangle rule exact to 2n+m."""
    q = (2 * n + m + 2) // 2
    lam, w = qd.tri_rule(q)
    Vn = eval_basis(n, lam)
    Vm = eval_basis(m, lam)
    Minv = np.array([[np.longdouble(x.numerator) / np.longdouble(x.denominator) for x in r] for r in mass_inv_exact(n)])
    P = Minv @ (Vn.T * (w * np.longdouble(2))[None, :])
    return Vn.astype(np.float64), Vm.astype(np.float64), P.astype(np.float64)


class OracleMesh2D:
    """Affine triangles: x = X0 + l1 (X1 - X0) + l2 (X2 - X0); edge f opposite vertex f, outward normals;
    neighbours matched by the sorted global vertex pair."""

    def __init__(self, vertices, elements):
        self.vertices = np.asarray(vertices, dtype=np.float64)
        self.elements = np.asarray(elements, dtype=np.int64)
        X = self.vertices[self.elements]
        self.X = X
        K = len(X)
        self.K = K
        E = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]], axis=-1)  # K, 2(x), 2(l)
        self.dxdr = E / 2.0
        self.J = np.linalg.det(self.dxdr)
        if np.any(self.J <= 0):
            raise ValueError("element with non-positive Jacobian (clockwise triangle)")
        self.G = np.linalg.inv(self.dxdr)  # G[k, ref, phys]
        self.Einv = np.linalg.inv(E)
        self.area = self.J * 2.0
        self.length = np.zeros((K, 3))
        self.normal = np.zeros((K, 3, 2))
        keys = {}
        for f in range(3):
            a, b = X[:, (f + 1) % 3], X[:, (f + 2) % 3]
            d = b - a
            self.length[:, f] = np.linalg.norm(d, axis=1)
            n = np.stack([d[:, 1], -d[:, 0]], axis=1) / self.length[:, f][:, None]
            sgn = np.sign(np.einsum("kd,kd->k", n, a - X[:, f]))
            self.normal[:, f] = n * sgn[:, None]
        self.nbr = -np.ones((K, 3), dtype=np.int64)
        for k in range(K):
            for f in range(3):
                key = tuple(sorted((int(self.elements[k, (f + 1) % 3]), int(self.elements[k, (f + 2) % 3]))))
                keys.setdefault(key, []).append((k, f))
        for v in keys.values():
            if len(v) > 2:
                raise ValueError("edge shared by more than two triangles")
            if len(v) == 2:
                (k1, f1), (k2, f2) = v
                self.nbr[k1, f1] = k2
                self.nbr[k2, f2] = k1

    def barycentric(self, k, x):
        l12 = np.einsum("kij,k...j->k...i", self.Einv[k], x - self.X[k, 0][:, None, :])
        return np.concatenate([1.0 - l12.sum(-1, keepdims=True), l12], axis=-1)


class Acoustic2DOracle:
    def __init__(self, vertices, elements, N: int, M: int, c2M, tau_p: float = 1.0, tau_u: float = 1.0,
                 source=None):
        self.mesh = vertices if isinstance(vertices, OracleMesh2D) else OracleMesh2D(vertices, elements)
        self.N, self.M = N, M
        self.Np = num_coeffs(N)
        self.tau_p, self.tau_u = float(tau_p), float(tau_u)
        c2M = np.asarray(c2M, dtype=np.float64)
        if c2M.shape != (self.mesh.K, num_coeffs(M)):
            raise ValueError("c2M must be [K, Np2(M)]")
        self.c2M = c2M
        self.D = derivative_ops(N)
        self.edge_lam, self.Vf, self.Lf = edge_ops(N)
        self.VqN, self.VqM, self.Pq = wadg_ops(N, M)
        self.c2q = c2M @ self.VqM.T
        self.source = None if source is None else np.asarray(source, dtype=np.float64)
        m = self.mesh
        self.edge_scale = m.length / m.area[:, None]
        # neighbour trace matrices at this element's physical edge points
        K = m.K
        nq = self.edge_lam[0].shape[0]
        self.Vnb = np.zeros((K, 3, nq, self.Np))
        for f in range(3):
            pts = np.einsum("qv,kvd->kqd", self.edge_lam[f], m.X)
            nb = m.nbr[:, f]
            ok = nb >= 0
            self.Vnb[ok, f] = eval_basis(N, m.barycentric(nb[ok], pts[ok]))

    def gradient(self, q):
        dref = np.einsum("dij,kj->kdi", self.D, q)
        return np.einsum("kdx,kdi->kxi", self.mesh.G, dref)

    def rhs_pre_wadg(self, Q, t: float = 0.0):
        m = self.mesh
        p, u = Q[:, 0], Q[:, 1:3]
        rp = -sum(self.gradient(u[:, c])[:, c] for c in range(2))
        ru = -self.gradient(p)
        for f in range(3):
            Vf = self.Vf[f]
            pm = p @ Vf.T
            um = np.einsum("qj,kcj->kcq", Vf, u)
            nb = m.nbr[:, f]
            inner = nb >= 0
            nbc = np.where(inner, nb, 0)
            pp = np.einsum("kqj,kj->kq", self.Vnb[:, f], p[nbc])
            up = np.einsum("kqj,kcj->kcq", self.Vnb[:, f], u[nbc])
            pp = np.where(inner[:, None], pp, -pm)
            up = np.where(inner[:, None, None], up, um)
            n = m.normal[:, f]
            jp = pp - pm
            jun = np.einsum("kc,kcq->kq", n, up - um)
            Fp = 0.5 * (self.tau_p * jp - jun)
            Fu = 0.5 * (self.tau_u * jun - jp)
            s = self.edge_scale[:, f][:, None]
            rp = rp + s * (Fp @ self.Lf[f].T)
            ru = ru + n[:, :, None] * (s * (Fu @ self.Lf[f].T))[:, None, :]
        if self.source is not None:
            rp = rp + self.source * np.sin(np.pi * t)
        return rp, ru

    def wadg(self, r):
        return ((r @ self.VqN.T) * self.c2q) @ self.Pq.T

    def rhs(self, Q, t: float = 0.0):
        rp, ru = self.rhs_pre_wadg(Q, t)
        out = np.empty_like(Q)
        out[:, 0] = self.wadg(rp)
        out[:, 1:3] = ru
        return out

    def step(self, Q, res, t, dt):
        for s in range(5):
            res *= float(LSRK_A[s])
            res += dt * self.rhs(Q, t + float(LSRK_C[s]) * dt)
            Q += float(LSRK_B[s]) * res
        return Q, res

    def run(self, Q0, t0, dt, nsteps):
        Q = np.array(Q0, dtype=np.float64, copy=True)
        res = np.zeros_like(Q)
        t = t0
        for _ in range(nsteps):
            self.step(Q, res, t, dt)
            t += dt
        return Q

    def energy(self, Q) -> float:
        """1/2 sum_k J_k [p^T M M_{c^2}^-1 M p + sum_i u_i^T M u_i] (R22 in 2D)."""
        Mh = mass(self.N)
        q = (2 * self.N + self.M + 2) // 2
        _, w = qd.tri_rule(q)
        wv = w.astype(np.float64) * 2.0
        Mp = Q[:, 0] @ Mh
        Mc = np.einsum("qi,kq,qj->kij", self.VqN, wv[None, :] * self.c2q, self.VqN)
        ep = np.einsum("ki,ki->k", Mp, np.linalg.solve(Mc, Mp[..., None])[..., 0])
        eu = np.einsum("kci,ij,kcj->k", Q[:, 1:3], Mh, Q[:, 1:3])
        return 0.5 * float(np.sum(self.mesh.J * (ep + eu)))

    def energy_rate(self, Q) -> float:
        Mh = mass(self.N)
        rp, ru = self.rhs_pre_wadg(Q)
        e = np.einsum("ki,ij,kj->k", Q[:, 0], Mh, rp) + np.einsum("kci,ij,kcj->k", Q[:, 1:3], Mh, ru)
        return float(np.sum(self.mesh.J * e))

    def l2_error(self, Q, exact, t, field: int = 0) -> float:
        lam, w = qd.tri_rule(self.N + 3)
        lam, w = lam.astype(np.float64), w.astype(np.float64)
        V = eval_basis(self.N, lam)
        pts = np.einsum("qv,kvd->kqd", lam, self.mesh.X)
        err = Q[:, field] @ V.T - exact(pts[..., 0], pts[..., 1], t)[field]
        return float(np.sqrt(np.sum(self.mesh.area[:, None] * w[None, :] * err * err)))
