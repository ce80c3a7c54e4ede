"""Bernstein basis on the reference tetrahedron (§2).

Reference tetrahedron D^ = {r,s,t >= -1, r+s+t <= -1} with vertices
v0=(-1,-1,-1), v1=(1,-1,-1), v2=(-1,1,-1), v3=(-1,-1,1) and barycentric
coordinates
    l0 = -(1+r+s+t)/2,  l1 = (1+r)/2,  l2 = (1+s)/2,  l3 = (1+t)/2.
B^N_a = N!/(a0! a1! a2! a3!) l0^a0 l1^a1 l2^a2 l3^a3, |a| = N.

Multi-index order: the ABI's canonical order (R19):
    for a3 in 0..N: for a2 in 0..N-a3: for a1 in 0..N-a3-a2:  a0 = N-a1-a2-a3.

Exact moments (used to build integer/rational reference matrices):
    int_T l^a dV = |T| d! prod(a_i!) / (|a| + d)!          (d = 3 volume, 2 face).
"""
from __future__ import annotations

import math
from fractions import Fraction
from functools import lru_cache

import numpy as np

REF_VOLUME = Fraction(4, 3)  # |D^| of the bi-unit reference tetrahedron
REF_VERTICES = np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])
# d(l_i)/d(r,s,t): rows i = 0..3, columns r,s,t
DLAMBDA_DREF = (
    (Fraction(-1, 2), Fraction(-1, 2), Fraction(-1, 2)),
    (Fraction(1, 2), Fraction(0), Fraction(0)),
    (Fraction(0), Fraction(1, 2), Fraction(0)),
    (Fraction(0), Fraction(0), Fraction(1, 2)),
)


def num_coeffs(n: int) -> int:
    """Np(n) = dim P^n on a tetrahedron = C(n+3, 3)."""
    return math.comb(n + 3, 3)


def num_face_coeffs(n: int) -> int:
    return math.comb(n + 2, 2)


@lru_cache(maxsize=None)
def multi_indices(n: int) -> tuple:
    out = []
    for a3 in range(n + 1):
        for a2 in range(n + 1 - a3):
            for a1 in range(n + 1 - a3 - a2):
                out.append((n - a1 - a2 - a3, a1, a2, a3))
    return tuple(out)


def multinomial(alpha) -> int:
    return math.factorial(sum(alpha)) // math.prod(math.factorial(a) for a in alpha)


def index_array(n: int) -> np.ndarray:
    return np.array(multi_indices(n), dtype=np.int64)


def eval_basis(n: int, lam: np.ndarray) -> np.ndarray:
    """B^n_a(lam) for barycentric points lam[..., 4]; returns [..., Np(n)].
    Works in the dtype of ``lam`` (float64 or longdouble)."""
    idx = index_array(n)
    C = np.array([multinomial(a) for a in multi_indices(n)], dtype=lam.dtype)
    return C * np.prod(lam[..., None, :] ** idx.astype(lam.dtype), axis=-1)


def barycentric_from_ref(rst: np.ndarray) -> np.ndarray:
    r, s, t = rst[..., 0], rst[..., 1], rst[..., 2]
    return np.stack([-(1 + r + s + t) / 2, (1 + r) / 2, (1 + s) / 2, (1 + t) / 2], axis=-1)


def simplex_moment(a, dim: int = 3) -> Fraction:
    """int over a simplex of measure 1 of prod l_i^a_i  =  d! prod a_i! / (|a|+d)!."""
    return Fraction(math.factorial(dim) * math.prod(math.factorial(x) for x in a), math.factorial(sum(a) + dim))


@lru_cache(maxsize=None)
def mass_integer(n: int):
    """Reference Bernstein mass matrix M^ = s * A with A integer:
    int B_a B_b = |T| C_a C_b 3! (a+b)! / (2n+3)!  =  |T| 6 (n!)^2/(2n+3)! * prod C(a_i+b_i, a_i).
    Returns (A as int64 numpy array, s as Fraction)."""
    idx = multi_indices(n)
    A = np.array([[math.prod(math.comb(a[i] + b[i], a[i]) for i in range(4)) for b in idx] for a in idx],
                 dtype=np.int64)
    s = REF_VOLUME * 6 * math.factorial(n) ** 2 / Fraction(math.factorial(2 * n + 3))
    return A, s


def mass_exact(n: int):
    """M^ as a list-of-lists of Fractions, straight from the moment formula."""
    idx = multi_indices(n)
    out = []
    for a in idx:
        row = []
        for b in idx:
            ab = tuple(x + y for x, y in zip(a, b))
            row.append(REF_VOLUME * multinomial(a) * multinomial(b) * simplex_moment(ab))
        out.append(row)
    return out


@lru_cache(maxsize=None)
def stiffness_exact(n: int, ref_dir: int):
    """S^_d[a,b] = int_{D^} B_a dB_b/d(ref_dir) dV, exact (Fractions), from
    dB_b/dr = sum_j (dl_j/dr) C_b b_j l^(b - e_j) and the moment formula.
    Returned as a numpy object array [Np, Np]."""
    idx = multi_indices(n)
    Np = len(idx)
    out = np.empty((Np, Np), dtype=object)
    for i, a in enumerate(idx):
        Ca = multinomial(a)
        for j, b in enumerate(idx):
            Cb = multinomial(b)
            acc = Fraction(0)
            for v in range(4):
                g = DLAMBDA_DREF[v][ref_dir]
                if g == 0 or b[v] == 0:
                    continue
                e = list(x + y for x, y in zip(a, b))
                e[v] -= 1
                acc += g * b[v] * simplex_moment(e)
            out[i, j] = REF_VOLUME * Ca * Cb * acc
    return out
