"""Elastic inputs: material coefficients and states -- data only.

State layout ``Q[K][9][Np]``: fields (v_1, v_2, v_3, s11, s22, s33, s23, s13, s12) (the Voigt order of
the rows of PAPER.md's A_i matrices).  Material inputs: per-element degree-M Bernstein
coefficients of rho^-1, lambda and mu (R25), arrays [K][Np(M)].

* random_material: parity inputs, Bernstein coefficients uniform in [0.5, 1.5] (rho^-1), [0.5, 1.5]
  (lambda), [0.25, 0.75] (mu): positive by the convex-hull property; numpy default_rng(809).
* smooth_material: rho^-1 = 1 + 1/4 sin(pi x) sin(pi y) sin(pi z), lambda = 1 + 1/2 sin(k pi x)..., mu =
  1/2 + 1/4 sin(k pi x)...  (the acoustic c^2 model of P:674 carried over to the Lame fields; the paper's
  elastic runs print no media -- DESIGN.md R25), L2-projected onto P^M.
* random_state: standard normal coefficients, default_rng(1809).
* standing_p_wave: the exact solution of DESIGN.md R27 (lambda = 0, mu = 1/2, rho = 1):
      v_i = cos(pi x_i) cos(pi t),  s_ii = -sin(pi x_i) sin(pi t),  shear stresses 0,
  traction-free on the faces of [-1,1]^3.
"""
from __future__ import annotations

from math import comb

import numpy as np

from ._l2fit import l2_fit

PARITY_MATERIAL_SEED = 809
PARITY_STATE_SEED = 1809
NFIELDS = 9


def num_coeffs(N: int) -> int:
    return comb(N + 3, 3)


def random_material(K: int, M: int, seed: int = PARITY_MATERIAL_SEED):
    rng = np.random.default_rng(seed)
    mp = num_coeffs(M)
    rho_inv = rng.uniform(0.5, 1.5, size=(K, mp))
    lam = rng.uniform(0.5, 1.5, size=(K, mp))
    mu = rng.uniform(0.25, 0.75, size=(K, mp))
    return rho_inv, lam, mu


def smooth_material(vertices, elements, M: int, k: float = 1.0, device=None):
    pi = np.pi

    def s3(x, y, z, kk, xp):
        return xp.sin(kk * pi * x) * xp.sin(kk * pi * y) * xp.sin(kk * pi * z)

    rho_inv = l2_fit(vertices, elements, lambda x, y, z, xp=np: 1.0 + 0.25 * s3(x, y, z, 1.0, xp), M, extra=4,
                     device=device)
    lam = l2_fit(vertices, elements, lambda x, y, z, xp=np: 1.0 + 0.5 * s3(x, y, z, k, xp), M, extra=4, device=device)
    mu = l2_fit(vertices, elements, lambda x, y, z, xp=np: 0.5 + 0.25 * s3(x, y, z, k, xp), M, extra=4, device=device)
    return rho_inv, lam, mu


def constant_material(K: int, M: int, rho_inv: float, lam: float, mu: float):
    """Constant fields: every Bernstein coefficient equals the value (partition of unity)."""
    mp = num_coeffs(M)
    return (np.full((K, mp), float(rho_inv)), np.full((K, mp), float(lam)), np.full((K, mp), float(mu)))


def random_state(K: int, N: int, seed: int = PARITY_STATE_SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((K, NFIELDS, num_coeffs(N)))


def standing_p_wave_exact(x, y, z, t, xp=np):
    pi = np.pi
    ct, st = np.cos(pi * t), np.sin(pi * t)
    zero = 0.0 * x
    return (xp.cos(pi * x) * ct, xp.cos(pi * y) * ct, xp.cos(pi * z) * ct,
            -xp.sin(pi * x) * st, -xp.sin(pi * y) * st, -xp.sin(pi * z) * st, zero, zero, zero)


def standing_p_wave_initial(vertices, elements, N: int, t: float = 0.0) -> np.ndarray:
    K = elements.shape[0]
    Q = np.zeros((K, NFIELDS, num_coeffs(N)))
    for c in range(6):
        Q[:, c, :] = l2_fit(vertices, elements, lambda x, y, z, c=c, xp=np: standing_p_wave_exact(x, y, z, t, xp)[c], N)
    return Q


def gaussian_pulse(vertices, elements, N: int, width: float = 50.0, device=None) -> np.ndarray:
    """Benchmark state: s11 = s22 = s33 = -exp(-width |x|^2) (a pressure pulse), v = 0, shear 0."""
    K = elements.shape[0]
    Q = np.zeros((K, NFIELDS, num_coeffs(N)))
    g = l2_fit(vertices, elements, lambda x, y, z, xp=np: xp.exp(-width * (x * x + y * y + z * z)), N, device=device)
    for c in (3, 4, 5):
        Q[:, c, :] = -g
    return Q
