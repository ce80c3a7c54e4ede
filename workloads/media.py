"""Wavespeed fields c^2(x) and their per-element degree-M Bernstein inputs.

* smooth / frequency-k:  c^2 = 1 + 1/2 sin(k pi x) sin(k pi y) sin(k pi z)
  (k=1; P:1051-1058 Eq. wavespeedk).
* layered (BASELINE.json config 4; no paper experiment -- DESIGN.md R23):
  c^2 = 1.0 (z < -0.3), 1.5 (-0.3 <= z < 0.35), 2.25 (z >= 0.35).
* random (parity inputs): Bernstein coefficients uniform in [0.5, 1.5]
  (positive by the convex-hull property), numpy default_rng(808).

The weight the WADG update multiplies by is c^2 (R1; PAPER.md Eq.
WADGform P:141), so these arrays are the c^2_M coefficients ``bbwadg_setup``
takes.
"""
from __future__ import annotations

import numpy as np

from ._l2fit import eval_at_rule, l2_fit

PARITY_C2_SEED = 808


def c2_smooth(k: float = 1.0):
    def f(x, y, z, xp=np):
        return 1.0 + 0.5 * xp.sin(k * np.pi * x) * xp.sin(k * np.pi * y) * xp.sin(k * np.pi * z)
    return f


def c2_layered(z0: float = -0.3, z1: float = 0.35, values=(1.0, 1.5, 2.25)):
    def f(x, y, z, xp=np):
        return xp.where(z < z0, values[0], xp.where(z < z1, values[1], values[2])) + 0.0 * x
    return f


def project_c2(vertices, elements, func, M: int, device=None) -> np.ndarray:
    """c^2_M: per-element L2 projection onto P^M (P:286 'quadrature-based L2
    projection') with q = M+4 points per direction (exact for polynomial
    integrands of degree 2M+7)."""
    return l2_fit(vertices, elements, func, M, extra=4, device=device)


def random_c2(K: int, M: int, seed: int = PARITY_C2_SEED, lo: float = 0.5, hi: float = 1.5) -> np.ndarray:
    from math import comb
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=(K, comb(M + 3, 3)))


def min_value(c2M: np.ndarray, M: int, q: int | None = None) -> float:
    """Minimum of c^2_M over a Stroud rule inside every element (input sanity)."""
    q = q if q is not None else M + 2
    return float(eval_at_rule(c2M, M, q).min())
