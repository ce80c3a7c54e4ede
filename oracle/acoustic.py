"""Oracle WADG acoustic solver (plain dense definitions, fp64 per element).

Semi-discrete scheme, Eq. WADGform with the sign reading of
DESIGN.md R3 (-volume + surface, as in Eq. matform P:120 / Eq. sdf):

  dp/dt   = (M^k)^-1 M^k_{c^2} [ -sum_ij G_ij D_j U_i + sum_f (J_f/J) L^f F_p  (+ Pi_N f) ]
  dU_i/dt = -sum_j G_ij D_j p + sum_f (J_f/J) n_i L^f F_u

with the penalty fluxes of Eq. sdf
  F_p = 1/2 (tau_p [[p]] - n.[[u]]),   F_u = 1/2 (tau_u [[u]].n - [[p]]),
  [[q]] = q+ - q,  n = outward normal of D^k;
boundary faces (R11): p+ = -p, u+ = u.
(M^k)^-1 M^k_{c^2} is applied as P_q diag(c^2_M(x_q)) V_q (Eq. pwadg, weight c^2
per DESIGN.md R1/R2).  The manufactured source enters as r_p += g sin(pi t)
before the projection (R17).

Time integration: 5-stage 2N-storage RK of Carpenter & Kennedy (P:1264
"low-storage 4th order Runge-Kutta method"; coefficients DESIGN.md R13):
  res = a_s res + dt rhs(Q, t + c_s dt);   Q = Q + b_s res.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from . import bernstein as bb
from . import operators as ops
from .mesh import OracleMesh

# Carpenter & Kennedy (1994) 5-stage, 4th-order, 2N-storage coefficients.
LSRK_A = (Fraction(0), Fraction(-567301805773, 1357537059087), Fraction(-2404267990393, 2016746695238),
          Fraction(-3550918686646, 2091501179385), Fraction(-1275806237668, 842570457699))
LSRK_B = (Fraction(1432997174477, 9575080441755), Fraction(5161836677717, 13612068292357),
          Fraction(1720146321549, 2090206949498), Fraction(3134564353537, 4481467310338),
          Fraction(2277821191437, 14882151754819))
LSRK_C = (Fraction(0), Fraction(1432997174477, 9575080441755), Fraction(2526269341429, 6820363962896),
          Fraction(2006345519317, 3224310063776), Fraction(2802321613138, 2924317926251))


class AcousticOracle:
    """Oracle for one mesh, degree N, material degree M and c^2_M coefficients."""

    def __init__(self, vertices, elements, N: int, M: int, c2M: np.ndarray,
                 tau_p: float = 1.0, tau_u: float = 1.0, source: np.ndarray | None = None):
        self.mesh = vertices if isinstance(vertices, OracleMesh) else OracleMesh(vertices, elements)
        self.N, self.M = N, M
        self.Np = bb.num_coeffs(N)
        self.tau_p, self.tau_u = float(tau_p), float(tau_u)
        c2M = np.asarray(c2M, dtype=np.float64)
        if c2M.shape != (self.mesh.K, bb.num_coeffs(M)):
            raise ValueError("c2M must be [K, Np(M)]")
        self.c2M = c2M
        self.D = ops.derivative_ops(N)  # 3,Np,Np
        self.face_lam, self.Vf, self.Lf = ops.face_ops(N)
        self.Vnb = self.mesh.neighbour_trace_matrices(N)
        self.VqN, self.VqM, self.Pq = ops.wadg_ops(N, M)
        self.c2q = c2M @ self.VqM.T  # K,nq: c^2_M at the WADG quadrature points
        self.source = None if source is None else np.asarray(source, dtype=np.float64)
        m = self.mesh
        self.face_scale = m.area / m.volume[:, None]  # |f|/|T|

    # ---- pieces of the right-hand side -------------------------------------------
    def gradient(self, q: np.ndarray) -> np.ndarray:
        """Physical gradient coefficients [K,3,Np] of fields q[K,Np]:
        d/dx_phys = sum_ref G[ref, phys] D_ref (chain rule)."""
        dref = np.einsum("dij,kj->kdi", self.D, q)
        return np.einsum("kdx,kdi->kxi", self.mesh.G, dref)

    def rhs_pre_wadg(self, Q: np.ndarray, t: float = 0.0):
        """(r_p, r_u): the bracket of Eq. WADGform before (M^k)^-1 M^k_{c^2}."""
        m = self.mesh
        p, u = Q[:, 0], Q[:, 1:4]
        rp = -sum(self.gradient(u[:, c])[:, c] for c in range(3))
        ru = -self.gradient(p)
        for f in range(4):
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
            n = m.normal[:, f]  # K,3
            jp = pp - pm
            jun = np.einsum("kc,kcq->kq", n, up - um)
            Fp = 0.5 * (self.tau_p * jp - jun)
            Fu = 0.5 * (self.tau_u * jun - jp)
            s = self.face_scale[:, f][:, None]
            lp = s * (Fp @ self.Lf[f].T)
            lu = s * (Fu @ self.Lf[f].T)
            rp = rp + lp
            ru = ru + n[:, :, None] * lu[:, None, :]
        if self.source is not None:
            rp = rp + self.source * np.sin(np.pi * t)
        return rp, ru

    def wadg(self, r: np.ndarray) -> np.ndarray:
        """(M^k)^-1 M^k_{c^2} r = P_q diag(c^2_M(x_q)) V_q r   (Eq. pwadg)."""
        return ((r @ self.VqN.T) * self.c2q) @ self.Pq.T

    def rhs(self, Q: np.ndarray, t: float = 0.0) -> np.ndarray:
        rp, ru = self.rhs_pre_wadg(Q, t)
        out = np.empty_like(Q)
        out[:, 0] = self.wadg(rp)
        out[:, 1:4] = ru
        return out

    # ---- time integration ----------------------------------------------------------
    def step(self, Q: np.ndarray, res: np.ndarray, t: float, dt: float):
        for s in range(5):
            res *= float(LSRK_A[s])
            res += dt * self.rhs(Q, t + float(LSRK_C[s]) * dt)
            Q += float(LSRK_B[s]) * res
        return Q, res

    def run(self, Q0: np.ndarray, t0: float, dt: float, nsteps: int):
        Q = np.array(Q0, dtype=np.float64, copy=True)
        res = np.zeros_like(Q)
        t = t0
        for _ in range(nsteps):
            self.step(Q, res, t, dt)
            t += dt
        return Q

    # ---- diagnostics ---------------------------------------------------------------
    def energy(self, Q: np.ndarray) -> float:
        """WADG energy 1/2 sum_k J_k [ p^T M M_{c^2}^-1 M p + sum_i u_i^T M u_i ]
        (the weight-adjusted norm that makes the scheme energy stable)."""
        Mh = ops.mass(self.N)
        _, w = ops.volume_rule(ops.wadg_quadrature_degree(self.N, self.M))
        wv = w * float(bb.REF_VOLUME)
        Mp = Q[:, 0] @ Mh  # K,Np (M symmetric)
        Mc = np.einsum("qi,kq,qj->kij", self.VqN, wv[None, :] * self.c2q, self.VqN)
        ep = np.einsum("ki,ki->k", Mp, np.linalg.solve(Mc, Mp[..., None])[..., 0])
        eu = np.einsum("kci,ij,kcj->k", Q[:, 1:4], Mh, Q[:, 1:4])
        return 0.5 * float(np.sum(self.mesh.J * (ep + eu)))

    def energy_rate(self, Q: np.ndarray) -> float:
        """Semi-discrete dE/dt = sum_k J_k [p^T M r_p + sum_i u_i^T M r_{u_i}]."""
        Mh = ops.mass(self.N)
        rp, ru = self.rhs_pre_wadg(Q)
        e = np.einsum("ki,ij,kj->k", Q[:, 0], Mh, rp) + np.einsum("kci,ij,kcj->k", Q[:, 1:4], Mh, ru)
        return float(np.sum(self.mesh.J * e))

    def l2_error(self, Q: np.ndarray, exact, t: float, field: int = 0, q: int | None = None) -> float:
        """||q_h - q||_{L2(Omega)} with a rule exact to degree >= 2N+2 (R18)."""
        q = q if q is not None else self.N + 3
        lam, w = ops.volume_rule(q)
        V = bb.eval_basis(self.N, lam)
        pts = np.einsum("qv,kvd->kqd", lam, self.mesh.X)
        ex = exact(pts[..., 0], pts[..., 1], pts[..., 2], t)[field]
        err = Q[:, field] @ V.T - ex
        return float(np.sqrt(np.sum(self.mesh.volume[:, None] * w[None, :] * err * err)))


def lsrk_stability_polynomial():
    """Coefficients (Fractions) of R(z) for y' = z y under one LSRK step of unit dt."""
    # represent y and res as polynomials in z (lists of Fractions)
    def add(a, b):
        n = max(len(a), len(b))
        return [(a[i] if i < len(a) else 0) + (b[i] if i < len(b) else 0) for i in range(n)]

    def scale(a, s):
        return [s * x for x in a]

    def shift(a):
        return [Fraction(0)] + list(a)

    y = [Fraction(1)]
    res = [Fraction(0)]
    for s in range(5):
        res = add(scale(res, LSRK_A[s]), shift(y))
        y = add(y, scale(res, LSRK_B[s]))
    return y
