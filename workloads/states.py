"""Initial states and manufactured-solution data (inputs only).

State layout (the ABI's canonical layout):
``Q[K][4][Np]`` float64, fields (p, u_x, u_y, u_z), Bernstein coefficients in
canonical multi-index order.

* random_state: standard normal coefficients, numpy default_rng(1808)
  (SURVEY.md §8d parity inputs).
* gaussian_pulse: p = exp(-50|x|^2), u = 0 (BASELINE config 3 state).
* manufactured (3D):
      p  =  sin(pi x) sin(pi y) sin(pi z) cos(pi t)
      u  = -(cos sin sin, sin cos sin, sin sin cos) sin(pi t)
      f  = (3 - 1/c^2) pi sin sin sin sin(pi t)
  The initial state is the L2 projection of (p, u) at t=0; the source data is
  g = Pi_N[(3 - 1/c^2) pi sin sin sin] so that the pressure source at time t is
  g * sin(pi t) (R17: added before the WADG projection).
"""
from __future__ import annotations

from math import comb

import numpy as np

from ._l2fit import l2_fit

PARITY_STATE_SEED = 1808


def num_coeffs(N: int) -> int:
    return comb(N + 3, 3)


def random_state(K: int, N: int, seed: int = PARITY_STATE_SEED) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal((K, 4, num_coeffs(N)))


def gaussian_pulse(vertices, elements, N: int, width: float = 50.0) -> np.ndarray:
    K = elements.shape[0]
    Q = np.zeros((K, 4, num_coeffs(N)))
    Q[:, 0, :] = l2_fit(vertices, elements, lambda x, y, z: np.exp(-width * (x * x + y * y + z * z)), N)
    return Q


def manufactured_exact(x, y, z, t, xp=np):
    s = xp.sin
    c = xp.cos
    pi = np.pi
    st, ct = np.sin(pi * t), np.cos(pi * t)
    p = s(pi * x) * s(pi * y) * s(pi * z) * ct
    ux = -c(pi * x) * s(pi * y) * s(pi * z) * st
    uy = -s(pi * x) * c(pi * y) * s(pi * z) * st
    uz = -s(pi * x) * s(pi * y) * c(pi * z) * st
    return p, ux, uy, uz


def manufactured_initial(vertices, elements, N: int, t: float = 0.0, device=None) -> np.ndarray:
    K = elements.shape[0]
    Q = np.zeros((K, 4, num_coeffs(N)))
    for c in range(4):
        Q[:, c, :] = l2_fit(vertices, elements, lambda x, y, z, c=c, xp=np: manufactured_exact(x, y, z, t, xp)[c], N,
                            device=device)
    return Q


def manufactured_source(vertices, elements, N: int, c2func, device=None) -> np.ndarray:
    """g[K][Np] with r_p += g * sin(pi t)."""
    pi = np.pi

    def f(x, y, z, xp=np):
        return (3.0 - 1.0 / c2func(x, y, z, xp=xp)) * pi * xp.sin(pi * x) * xp.sin(pi * y) * xp.sin(pi * z)

    return l2_fit(vertices, elements, f, N, device=device)
