"""Extended-precision simplex quadrature (oracle tables only).

Collapsed-coordinate (Stroud conical product) rules -- the rule the paper
switches to for N > 7 ("collapsed coordinate
quadrature"); R15 uses it at every N with exactness >= 2N+M so that
quadrature WADG (Eq. pwadg) is exact for the polynomial weight c^2_M.

Nodes/weights are computed by mpmath at 40 digits and returned as numpy
``longdouble`` (80-bit) arrays, so that rule error does not get amplified by
the Bernstein mass-matrix condition number.

Unit simplex {x,y,z >= 0, x+y+z <= 1}:  x = u, y = v(1-u), z = w(1-u)(1-v),
dV = (1-u)^2 (1-v) du dv dw; Gauss-Jacobi (2,0) in u, (1,0) in v, Legendre in w.
q points per direction integrate polynomials of total degree <= 2q-1 exactly.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np
from mpmath import mp

DPS = 40


def _to_ld(values) -> np.ndarray:
    return np.array([np.longdouble(mp.nstr(v, 30, strip_zeros=False)) for v in values], dtype=np.longdouble)


@lru_cache(maxsize=None)
def gauss_jacobi01(q: int, alpha: int):
    """Nodes on [0,1] and weights for int_0^1 (1-u)^alpha g(u) du (mpmath mpf)."""
    with mp.workdps(DPS):
        X, W = mp.gauss_quadrature(q, "jacobi", alpha, 0)
        u = [(x + 1) / 2 for x in X]
        w = [wk / mp.mpf(2) ** (alpha + 1) for wk in W]
    return u, w


@lru_cache(maxsize=None)
def tet_rule(q: int):
    """Barycentric points [q^3, 4] (longdouble) and weights (longdouble) that
    sum to 1 (i.e. int_T g = |T| * sum w_i g(x_i))."""
    u, wu = gauss_jacobi01(q, 2)
    v, wv = gauss_jacobi01(q, 1)
    w, ww = gauss_jacobi01(q, 0)
    lam, wt = [], []
    with mp.workdps(DPS):
        for i in range(q):
            for j in range(q):
                for k in range(q):
                    x = u[i]
                    y = v[j] * (1 - u[i])
                    z = w[k] * (1 - u[i]) * (1 - v[j])
                    lam.append((1 - x - y - z, x, y, z))
                    wt.append(wu[i] * wv[j] * ww[k] * 6)
        lam_ld = _to_ld([c for p in lam for c in p]).reshape(-1, 4)
        wt_ld = _to_ld(wt)
    return lam_ld, wt_ld


@lru_cache(maxsize=None)
def tri_rule(q: int):
    """Triangle rule: barycentrics [q^2, 3] and weights summing to 1."""
    u, wu = gauss_jacobi01(q, 1)
    v, wv = gauss_jacobi01(q, 0)
    lam, wt = [], []
    with mp.workdps(DPS):
        for i in range(q):
            for j in range(q):
                x = u[i]
                y = v[j] * (1 - u[i])
                lam.append((1 - x - y, x, y))
                wt.append(wu[i] * wv[j] * 2)
        lam_ld = _to_ld([c for p in lam for c in p]).reshape(-1, 3)
        wt_ld = _to_ld(wt)
    return lam_ld, wt_ld


def face_rule(q: int, f: int):
    """Rule on reference face f (the face opposite vertex f, l_f = 0), as
    tetrahedron barycentrics [nq, 4]; the face's three vertices (increasing
    local index) take the triangle barycentrics in order.  Weights sum to 1."""
    lam3, wt = tri_rule(q)
    lam = np.zeros((lam3.shape[0], 4), dtype=np.longdouble)
    others = [v for v in range(4) if v != f]
    for c, v in enumerate(others):
        lam[:, v] = lam3[:, c]
    return lam, wt
