"""2D inputs ("2D triangles"; 2D experiments P:646-660, Fig. con2d
P:685-847) -- data only, no hot-path arithmetic.

* tri_mesh(n): [-1,1]^2 cut into n x n squares, each split into 2 triangles along its (0,0)-(1,1) diagonal,
  squares in Morton order, vertices counter-clockwise (positive orientation of the reference triangle
  {r, s >= -1, r + s <= 0}, vertices (-1,-1), (1,-1), (-1,1)).  K = 2 n^2.
* c2_smooth_2d(k): c^2 = 1 + 1/2 sin(k pi x) sin(k pi y) (k = 1), and per-element L2 fits to P^M.
* states: random coefficients (rng 2808), the 2D manufactured solution of P:646-652
      p = sin(pi x) sin(pi y) cos(pi t),  u = -(cos(pi x) sin(pi y), sin(pi x) cos(pi y)) sin(pi t),
      f = (2 - 1/c^2) pi sin(pi x) sin(pi y) sin(pi t)   (source g = Pi_N[(2 - 1/c^2) pi sin sin], r_p += g sin(pi t)),
  and a Gaussian pressure pulse.
State layout Q[K][3][Np2], Np2 = (N+1)(N+2)/2, fields (p, u_x, u_y), canonical order
``for a2 in 0..N: for a1 in 0..N-a2: a0 = N - a1 - a2`` (R29).
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np
from scipy.special import roots_jacobi

PARITY_STATE_SEED_2D = 2808
PARITY_C2_SEED_2D = 2809


def num_coeffs(N: int) -> int:
    return (N + 1) * (N + 2) // 2


def _morton2(i, j):
    out = np.zeros_like(i)
    for b in range(16):
        out |= ((i >> b) & 1) << (2 * b)
        out |= ((j >> b) & 1) << (2 * b + 1)
    return out


def tri_mesh(n: int):
    """(vertices [nv, 2], triangles [2 n^2, 3] int64)."""
    xs = np.linspace(-1.0, 1.0, n + 1)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    V = np.stack([X.ravel(), Y.ravel()], axis=1)
    vid = lambda i, j: i * (n + 1) + j  # noqa: E731
    I, J = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    I, J = I.ravel(), J.ravel()
    order = np.argsort(_morton2(I, J), kind="stable")
    I, J = I[order], J[order]
    v00, v10, v01, v11 = vid(I, J), vid(I + 1, J), vid(I, J + 1), vid(I + 1, J + 1)
    T = np.empty((2 * len(I), 3), dtype=np.int64)
    T[0::2] = np.stack([v00, v10, v11], axis=1)  # lower-right triangle, counter-clockwise
    T[1::2] = np.stack([v00, v11, v01], axis=1)  # upper-left triangle, counter-clockwise
    return V, T


def min_height(vertices, elements) -> float:
    X = vertices[elements]
    h = np.inf
    for f in range(3):
        a, b = X[:, (f + 1) % 3], X[:, (f + 2) % 3]
        c = X[:, f]
        area2 = np.abs((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0]))
        h = min(h, float(np.min(area2 / np.linalg.norm(b - a, axis=1))))
    return h


@lru_cache(maxsize=None)
def _indices(n):
    return np.array([(n - a1 - a2, a1, a2) for a2 in range(n + 1) for a1 in range(n + 1 - a2)], dtype=np.int64)


@lru_cache(maxsize=None)
def _rule(q):
    """Collapsed Gauss-Jacobi rule on the unit triangle, exact to degree 2q-1; barycentric points, weights sum 1."""
    xu, wu = roots_jacobi(q, 1.0, 0.0)
    xv, wv = roots_jacobi(q, 0.0, 0.0)
    u, v = (xu + 1) / 2, (xv + 1) / 2
    U, Vv = np.meshgrid(u, v, indexing="ij")
    WU, WV = np.meshgrid(wu / 4.0, wv / 2.0, indexing="ij")
    x, y = U.ravel(), (Vv * (1 - U)).ravel()
    return np.stack([1 - x - y, x, y], axis=1), (WU * WV).ravel() * 2.0


def _basis(n, lam):
    idx = _indices(n)
    C = np.array([math.factorial(n) // math.prod(math.factorial(a) for a in al) for al in idx], dtype=np.float64)
    return C * np.prod(lam[..., None, :] ** idx, axis=-1)


@lru_cache(maxsize=None)
def _fit_op(n, q):
    lam, w = _rule(q)
    V = _basis(n, lam)
    return lam, np.linalg.solve(V.T @ (w[:, None] * V), V.T * w[None, :])


def l2_fit(vertices, elements, func, degree: int, extra: int = 4) -> np.ndarray:
    """Bernstein coefficients [K, Np2(degree)] of the per-element L2 projection of func(x, y)."""
    lam, P = _fit_op(degree, degree + extra)
    out = np.empty((len(elements), P.shape[0]))
    for s in range(0, len(elements), 65536):
        X = vertices[elements[s:s + 65536]]  # c,3,2
        pts = np.einsum("qv,kvd->kqd", lam, X)
        out[s:s + 65536] = func(pts[..., 0], pts[..., 1]) @ P.T
    return out


def c2_smooth_2d(k: float = 1.0):
    return lambda x, y: 1.0 + 0.5 * np.sin(k * np.pi * x) * np.sin(k * np.pi * y)


def project_c2(vertices, elements, func, M: int) -> np.ndarray:
    return l2_fit(vertices, elements, func, M)


def random_c2(K: int, M: int, seed: int = PARITY_C2_SEED_2D) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.5, 1.5, size=(K, num_coeffs(M)))


def random_state(K: int, N: int, seed: int = PARITY_STATE_SEED_2D) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((K, 3, num_coeffs(N)))


def manufactured_exact(x, y, t):
    s, c, pi = np.sin, np.cos, np.pi
    st, ct = np.sin(pi * t), np.cos(pi * t)
    return (s(pi * x) * s(pi * y) * ct, -c(pi * x) * s(pi * y) * st, -s(pi * x) * c(pi * y) * st)


def manufactured_initial(vertices, elements, N: int) -> np.ndarray:
    Q = np.zeros((len(elements), 3, num_coeffs(N)))
    for c in range(3):
        Q[:, c] = l2_fit(vertices, elements, lambda x, y, c=c: manufactured_exact(x, y, 0.0)[c], N)
    return Q


def manufactured_source(vertices, elements, N: int, c2func) -> np.ndarray:
    pi = np.pi
    return l2_fit(vertices, elements,
                  lambda x, y: (2.0 - 1.0 / c2func(x, y)) * pi * np.sin(pi * x) * np.sin(pi * y), N)


def gaussian_pulse(vertices, elements, N: int, width: float = 50.0) -> np.ndarray:
    Q = np.zeros((len(elements), 3, num_coeffs(N)))
    Q[:, 0] = l2_fit(vertices, elements, lambda x, y: np.exp(-width * (x * x + y * y)), N)
    return Q
