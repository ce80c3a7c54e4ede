"""Per-element least-squares (L2) fits of functions to Bernstein coefficients.

Input preparation only (see package docstring): this turns analytic fields
(wavespeed c^2, initial pressure, manufactured source) into the per-element
Bernstein coefficient arrays the hot path consumes.  fp64, Stroud conical
product rule from scipy's Gauss-Jacobi nodes, weighted least squares.  The
results are DATA handed identically to the oracle and to the CUDA library; their
accuracy (~1e-12 at N=9) is far below any discretisation error they feed.
"""
from __future__ import annotations

import math
from functools import lru_cache

import numpy as np
from scipy.special import roots_jacobi


@lru_cache(maxsize=None)
def _indices(n: int):
    out = []
    for a3 in range(n + 1):
        for a2 in range(n + 1 - a3):
            for a1 in range(n + 1 - a3 - a2):
                out.append((n - a1 - a2 - a3, a1, a2, a3))
    return np.array(out, dtype=np.int64)


@lru_cache(maxsize=None)
def _rule(q: int):
    """Collapsed-coordinate rule on the unit simplex, exact to degree 2q-1.
    Returns barycentric points [nq,4] and weights summing to 1."""
    xu, wu = roots_jacobi(q, 2.0, 0.0)
    xv, wv = roots_jacobi(q, 1.0, 0.0)
    xw, ww = roots_jacobi(q, 0.0, 0.0)
    u, v, w = (xu + 1) / 2, (xv + 1) / 2, (xw + 1) / 2
    wu, wv, ww = wu / 8.0, wv / 4.0, ww / 2.0
    U, V, W = np.meshgrid(u, v, w, indexing="ij")
    WU, WV, WW = np.meshgrid(wu, wv, ww, indexing="ij")
    x = U
    y = V * (1 - U)
    z = W * (1 - U) * (1 - V)
    lam = np.stack([1 - x - y - z, x, y, z], axis=-1).reshape(-1, 4)
    wt = (WU * WV * WW).reshape(-1) * 6.0
    return lam, wt


def _basis(n: int, lam: np.ndarray) -> np.ndarray:
    idx = _indices(n)
    C = np.array([math.factorial(n) // math.prod(math.factorial(a) for a in al) for al in idx], dtype=np.float64)
    return C * np.prod(lam[..., None, :] ** idx, axis=-1)


@lru_cache(maxsize=None)
def _fit_operator(n: int, q: int):
    lam, wt = _rule(q)
    V = _basis(n, lam)
    A = V.T @ (wt[:, None] * V)
    P = np.linalg.solve(A, V.T * wt[None, :])  # [Np, nq]
    return lam, P


def l2_fit(vertices: np.ndarray, elements: np.ndarray, func, degree: int, extra: int = 4,
           chunk: int = 65536, device=None) -> np.ndarray:
    """Bernstein coefficients [K, Np(degree)] of the per-element L2 projection
    of ``func(x, y, z)`` (vectorised; numpy or torch ufuncs via ``xp=``) onto
    P^degree, canonical index order.  ``device="cuda"`` evaluates with torch
    (fp64) on the GPU -- input synthesis for million-element meshes only."""
    q = degree + extra
    lam, P = _fit_operator(degree, q)
    K = elements.shape[0]
    out = np.empty((K, P.shape[0]), dtype=np.float64)
    if device is not None:
        import torch

        lam_t = torch.from_numpy(lam).to(device)
        P_t = torch.from_numpy(P).to(device)
        V_t = torch.from_numpy(vertices).to(device)
        chunk = max(1024, int(6e7 // lam.shape[0]))  # ~0.5 GB of fp64 points per chunk
        for s in range(0, K, chunk):
            E_t = torch.from_numpy(elements[s:s + chunk]).to(device)
            pts = torch.einsum("qv,cvd->cqd", lam_t, V_t[E_t])
            fv = func(pts[..., 0], pts[..., 1], pts[..., 2], xp=torch)
            out[s:s + chunk] = (fv @ P_t.T).cpu().numpy()
        return out
    for s in range(0, K, chunk):
        X = vertices[elements[s:s + chunk]]  # c,4,3
        pts = np.einsum("qv,cvd->cqd", lam, X)
        fv = func(pts[..., 0], pts[..., 1], pts[..., 2])
        out[s:s + chunk] = fv @ P.T
    return out


def eval_at_rule(coeffs: np.ndarray, degree: int, q: int):
    """Values of per-element Bernstein polynomials at the rule points (for
    positivity checks of inputs)."""
    lam, _ = _rule(q)
    return coeffs @ _basis(degree, lam).T
