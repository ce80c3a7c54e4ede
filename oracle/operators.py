"""Dense reference-element operators of the WADG scheme (oracle).

All operators are the paper's plain dense definitions:

* D_d   = M^-1 S_d                     (d = r,s,t reference directions)
* L'_f  = |T^| M^-1 V_f^T diag(w_f)     (lift L^f = M^-1 M_f of P:146 applied by
                                         face quadrature; w_f sums to 1, so that
                                         (M^k)^-1 int_f F phi = (|f|/|T|) L'_f F(x_q))
* P_q   = M^-1 V_q^T diag(w |T^|)       (Eq. pwadg)

"M^-1 X" is computed as the solution of M Y = X by mixed-precision iterative
refinement: M = s*A with A an exact integer matrix (``bernstein.mass_integer``),
fp64 Cholesky corrections, longdouble (80-bit) residuals, longdouble
right-hand sides from exact rationals or 40-digit quadrature.  The result is
rounded to fp64 once.  cond(M_9) ~ 3e5, so a plain fp64 solve would carry
~1e-12 errors into the oracle; refinement brings the
tables to ~1e-16 (pinned in tests/test_oracle_operators.py).
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache

import numpy as np
import scipy.linalg as sla
from mpmath import mp

from . import bernstein as bb
from . import quadrature as qd

LD = np.longdouble


def frac_to_ld(x: Fraction) -> np.longdouble:
    with mp.workdps(40):
        return np.longdouble(mp.nstr(mp.mpf(x.numerator) / x.denominator, 30, strip_zeros=False))


def mass_solve(n: int, rhs_ld: np.ndarray, iters: int = 4) -> np.ndarray:
    """Solve M^_n Y = rhs (rhs longdouble [Np, m]); returns Y in longdouble."""
    A, s = bb.mass_integer(n)
    rhs = rhs_ld / frac_to_ld(s)
    cho = sla.cho_factor(A.astype(np.float64))
    A_ld = A.astype(LD)
    Y = sla.cho_solve(cho, rhs.astype(np.float64)).astype(LD)
    for _ in range(iters):
        res = rhs - A_ld @ Y
        Y = Y + sla.cho_solve(cho, res.astype(np.float64)).astype(LD)
    return Y


@lru_cache(maxsize=None)
def mass(n: int) -> np.ndarray:
    """M^_n in fp64 (rounded once from the exact rational matrix)."""
    A, s = bb.mass_integer(n)
    return (A.astype(LD) * frac_to_ld(s)).astype(np.float64)


@lru_cache(maxsize=None)
def derivative_ops(n: int) -> np.ndarray:
    """D_r, D_s, D_t = M^-1 S_d, fp64 [3, Np, Np]."""
    out = []
    for d in range(3):
        S = bb.stiffness_exact(n, d)
        S_ld = np.array([[frac_to_ld(x) for x in row] for row in S], dtype=LD)
        out.append(mass_solve(n, S_ld).astype(np.float64))
    return np.stack(out)


def face_quadrature_degree(n: int) -> int:
    # the flux F (degree n on the face) times a test function (degree n): 2n
    return n + 1


@lru_cache(maxsize=None)
def face_ops(n: int):
    """Per reference face f = 0..3: barycentric face points lam_f [nq,4] (fp64),
    trace evaluation V_f [nq, Np] (fp64) and the lift L'_f [Np, nq] (fp64)."""
    q = face_quadrature_degree(n)
    lams, Vs, Ls = [], [], []
    vol_ld = frac_to_ld(bb.REF_VOLUME)
    for f in range(4):
        lam, w = qd.face_rule(q, f)
        V = bb.eval_basis(n, lam)  # longdouble
        L = mass_solve(n, V.T * (w * vol_ld)[None, :])
        lams.append(lam.astype(np.float64))
        Vs.append(V.astype(np.float64))
        Ls.append(L.astype(np.float64))
    return lams, Vs, Ls


def wadg_quadrature_degree(n: int, m: int) -> int:
    """q with 2q-1 >= 2n+m (Eq. pwadg exact for the degree-m weight)."""
    return (2 * n + m + 2) // 2


@lru_cache(maxsize=None)
def wadg_ops(n: int, m: int):
    """Quadrature WADG tables (Eq. pwadg): V_q^n [nq, Np(n)], V_q^m [nq, Np(m)],
    P_q [Np(n), nq] = M^-1 V_q^T diag(w |T^|), fp64."""
    q = wadg_quadrature_degree(n, m)
    lam, w = qd.tet_rule(q)
    Vn = bb.eval_basis(n, lam)
    Vm = bb.eval_basis(m, lam)
    P = mass_solve(n, Vn.T * (w * frac_to_ld(bb.REF_VOLUME))[None, :])
    return Vn.astype(np.float64), Vm.astype(np.float64), P.astype(np.float64)


@lru_cache(maxsize=None)
def volume_rule(q: int):
    lam, w = qd.tet_rule(q)
    return lam.astype(np.float64), w.astype(np.float64)
