"""L2 error of a per-element Bernstein field against an analytic function (output evaluation).

Used by the config-2 convergence study (BASELINE.json configs[1]; R18: the error is
||p_h(T) - p(T)||_{L2(Omega)} with a rule exact to >= 2N+2).  Like the rest of ``workloads`` it holds
none of the hot path's arithmetic: it evaluates the Bernstein expansion at the points of a
collapsed-coordinate (Stroud) rule exact to degree 2N+7 and integrates the squared difference with
the element Jacobians.
"""
from __future__ import annotations

import numpy as np

from ._l2fit import _basis, _rule


def l2_error(vertices: np.ndarray, elements: np.ndarray, coeffs: np.ndarray, degree: int, func,
             q: int | None = None, chunk: int = 65536) -> float:
    """sqrt(sum_k int_{T_k} (sum_a coeffs[k,a] B_a - func)^2) for coeffs [K, Np(degree)]; q points per
    direction (default degree + 4: exact to 2 degree + 7, well above R18's 2N+2, since func is not a
    polynomial)."""
    lam, wt = _rule(q if q is not None else degree + 4)
    V = _basis(degree, lam)  # [nq, Np]
    total = 0.0
    for s in range(0, elements.shape[0], chunk):
        el = elements[s:s + chunk]
        X = vertices[el]  # [k, 4, 3]
        pts = np.einsum("qv,kvd->kqd", lam, X)
        vol = np.abs(np.linalg.det(X[:, 1:] - X[:, :1])) / 6.0
        diff = coeffs[s:s + chunk] @ V.T - func(pts[..., 0], pts[..., 1], pts[..., 2])
        total += float(np.sum(vol[:, None] * wt[None, :] * diff * diff))
    return float(np.sqrt(total))
