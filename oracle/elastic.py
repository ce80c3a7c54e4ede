"""Oracle WADG elastic solver (plain dense definitions, fp64 per element) -- TEST INFRASTRUCTURE.

First-order velocity-stress elastic wave equation, Eq. ewave:
    rho dv/dt      = sum_i A_i^T d sigma/dx_i
    C^-1 dsigma/dt = sum_i A_i   d v/dx_i
with v = (v_1, v_2, v_3), sigma = (s11, s22, s33, s23, s13, s12) (Voigt order of the A_i rows,
P:159-183) and the isotropic C of P:185-195 (lambda + 2 mu, lambda on the normal block, mu I on the
shear block).  State Q[K][9][Np]: fields (v_1, v_2, v_3, s11, s22, s33, s23, s13, s12).

Semi-discrete scheme: the strong form of the elastic DG formulation, with its penalty
fluxes, [[q]] = q+ - q, n the outward normal of D^k, A_n = sum_i n_i A_i:
    F_v     = 1/2 A_n^T [[sigma]] + tau_v/2 A_n^T A_n [[v]]
    F_sigma = 1/2 A_n   [[v]]     + tau_s/2 A_n A_n^T [[sigma]]
    r_v     = sum_i A_i^T D_{x_i} sigma + sum_f (J_f/J) L^f F_v
    r_sigma = sum_i A_i   D_{x_i} v     + sum_f (J_f/J) L^f F_sigma
and the matrix-weighted WADG update of Eq. ewadg:
    dV/dt     = (I x M^-1) M_{rho^-1 I} r_v      -> per component P_q diag(rho^-1(x_q)) V_q r_{v,a}
    dSigma/dt = (I x M^-1) M_C r_sigma           -> (dSigma/dt)_s = sum_t P_q diag(C_st(x_q)) V_q r_{sigma,t}
(M_{C} is the block matrix of scalar weighted mass matrices M_{C_st}; each block applied
by the quadrature form of Eq. pwadg, exact for the degree-M polynomial weights).
Boundary faces (R26): traction-free mirror sigma+ = -sigma, v+ = v (the elastic analogue
of the acoustic pressure-release R11; with it {{A_n^T sigma}} = 0 on the boundary).
Material inputs (R25): per-element degree-M Bernstein coefficients of rho^-1, lambda, mu.

Pins: tests/test_oracle_elastic.py (linear-field exactness of the volume terms, constant-weight WADG
= C r, the mu = 0 / rho = 1 reduction to the (pinned) acoustic oracle, the energy-rate identity with
the penalty face integrals, energy conservation with tau = 0, and the convergence rate on the exact
standing P-wave of DESIGN.md R27).
"""
from __future__ import annotations

import numpy as np

from . import bernstein as bb
from . import operators as ops
from .acoustic import LSRK_A, LSRK_B, LSRK_C
from .mesh import OracleMesh

# A_1, A_2, A_3 of P:159-183 (6 x 3): rows = (s11, s22, s33, s23, s13, s12), columns = (v1, v2, v3)
A_MATS = np.zeros((3, 6, 3))
A_MATS[0, 0, 0] = 1.0
A_MATS[0, 4, 2] = 1.0
A_MATS[0, 5, 1] = 1.0
A_MATS[1, 1, 1] = 1.0
A_MATS[1, 3, 2] = 1.0
A_MATS[1, 5, 0] = 1.0
A_MATS[2, 2, 2] = 1.0
A_MATS[2, 3, 1] = 1.0
A_MATS[2, 4, 0] = 1.0


def isotropic_C(lam: np.ndarray, mu: np.ndarray) -> np.ndarray:
    """C[..., 6, 6] of P:185-195 from Lame parameters lam, mu (any broadcastable shape)."""
    lam = np.asarray(lam, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    C = np.zeros(np.broadcast(lam, mu).shape + (6, 6))
    for s in range(3):
        for t in range(3):
            C[..., s, t] = lam + (2.0 * mu if s == t else 0.0)
    for s in range(3, 6):
        C[..., s, s] = mu
    return C


class ElasticOracle:
    """Oracle for one mesh, degree N, material degree M, coefficients of rho^-1, lambda, mu."""

    def __init__(self, vertices, elements, N: int, M: int, rho_inv: np.ndarray, lam: np.ndarray, mu: np.ndarray,
                 tau_v: float = 1.0, tau_s: float = 1.0):
        self.mesh = vertices if isinstance(vertices, OracleMesh) else OracleMesh(vertices, elements)
        self.N, self.M = N, M
        self.Np = bb.num_coeffs(N)
        self.tau_v, self.tau_s = float(tau_v), float(tau_s)
        Mp = bb.num_coeffs(M)
        mats = []
        for a in (rho_inv, lam, mu):
            a = np.asarray(a, dtype=np.float64)
            if a.shape != (self.mesh.K, Mp):
                raise ValueError("material coefficients must be [K, Np(M)]")
            mats.append(a)
        self.rho_inv, self.lam, self.mu = mats
        self.D = ops.derivative_ops(N)
        self.face_lam, self.Vf, self.Lf = ops.face_ops(N)
        self.Vnb = self.mesh.neighbour_trace_matrices(N)
        self.VqN, self.VqM, self.Pq = ops.wadg_ops(N, M)
        # material at the WADG quadrature points
        self.rho_inv_q = self.rho_inv @ self.VqM.T  # K,nq
        self.Cq = isotropic_C(self.lam @ self.VqM.T, self.mu @ self.VqM.T)  # K,nq,6,6
        self.face_scale = self.mesh.area / self.mesh.volume[:, None]

    def gradient(self, q: np.ndarray) -> np.ndarray:
        """Physical gradient coefficients [K,3,Np] of fields q[K,Np] (chain rule)."""
        dref = np.einsum("dij,kj->kdi", self.D, q)
        return np.einsum("kdx,kdi->kxi", self.mesh.G, dref)

    def rhs_pre_wadg(self, Q: np.ndarray):
        """(r_v [K,3,Np], r_sigma [K,6,Np]): the brackets of Eq. ewadg before the WADG mass inverses."""
        m = self.mesh
        v, sg = Q[:, 0:3], Q[:, 3:9]
        gv = np.stack([self.gradient(v[:, a]) for a in range(3)], axis=1)  # K,3(a),3(x),Np
        gs = np.stack([self.gradient(sg[:, s]) for s in range(6)], axis=1)  # K,6(s),3(x),Np
        # volume: sum_i A_i^T d_i sigma, sum_i A_i d_i v
        rv = np.einsum("isa,ksin->kan", A_MATS, gs)
        rs = np.einsum("isa,kain->ksn", A_MATS, gv)
        for f in range(4):
            Vf = self.Vf[f]
            vm = np.einsum("qj,kcj->kcq", Vf, v)
            sm = np.einsum("qj,kcj->kcq", Vf, sg)
            nb = m.nbr[:, f]
            inner = nb >= 0
            nbc = np.where(inner, nb, 0)
            vp = np.einsum("kqj,kcj->kcq", self.Vnb[:, f], v[nbc])
            sp = np.einsum("kqj,kcj->kcq", self.Vnb[:, f], sg[nbc])
            vp = np.where(inner[:, None, None], vp, vm)
            sp = np.where(inner[:, None, None], sp, -sm)
            An = np.einsum("ki,isa->ksa", m.normal[:, f], A_MATS)  # K,6,3
            jv, js = vp - vm, sp - sm
            Fv = 0.5 * np.einsum("ksa,ksq->kaq", An, js) + 0.5 * self.tau_v * np.einsum(
                "ksa,ksb,kbq->kaq", An, An, jv)
            Fs = 0.5 * np.einsum("ksa,kaq->ksq", An, jv) + 0.5 * self.tau_s * np.einsum(
                "ksa,kta,ktq->ksq", An, An, js)
            s = self.face_scale[:, f][:, None, None]
            rv = rv + s * np.einsum("kaq,nq->kan", Fv, self.Lf[f])
            rs = rs + s * np.einsum("ksq,nq->ksn", Fs, self.Lf[f])
        return rv, rs

    def wadg_v(self, r: np.ndarray) -> np.ndarray:
        """(M^k)^-1 M^k_{rho^-1} applied to r[K,Np] (Eq. pwadg with weight rho^-1)."""
        return ((r @ self.VqN.T) * self.rho_inv_q) @ self.Pq.T

    def wadg_sigma(self, r: np.ndarray) -> np.ndarray:
        """(I x M^-1) M_C applied to r[K,6,Np]: out_s = sum_t P_q diag(C_st(x_q)) V_q r_t."""
        rq = np.einsum("qn,ktn->ktq", self.VqN, r)
        return np.einsum("kqst,ktq,nq->ksn", self.Cq, rq, self.Pq)

    def rhs(self, Q: np.ndarray, t: float = 0.0) -> np.ndarray:
        rv, rs = self.rhs_pre_wadg(Q)
        out = np.empty_like(Q)
        for a in range(3):
            out[:, a] = self.wadg_v(rv[:, a])
        out[:, 3:9] = self.wadg_sigma(rs)
        return out

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
        """WADG energy 1/2 sum_k J_k [ sum_a v_a^T M M_{rho^-1}^-1 M v_a + Sigma^T (IxM) M_C^-1 (IxM) Sigma ]
        (the weight-adjusted norm of Eq. ewadg, the inverse of its mass-inverse approximation)."""
        Mh = ops.mass(self.N)
        _, w = ops.volume_rule(ops.wadg_quadrature_degree(self.N, self.M))
        wv = w * float(bb.REF_VOLUME)
        Np = self.Np
        Mr = np.einsum("qi,kq,qj->kij", self.VqN, wv[None, :] * self.rho_inv_q, self.VqN)
        MV = np.einsum("kan,nm->kam", Q[:, 0:3], Mh)
        ev = np.einsum("kan,kan->k", MV, np.linalg.solve(Mr[:, None], MV[..., None])[..., 0])
        MC = np.einsum("qi,kqst,q,qj->ksitj", self.VqN, self.Cq, wv, self.VqN).reshape(-1, 6 * Np, 6 * Np)
        MS = np.einsum("ksn,nm->ksm", Q[:, 3:9], Mh).reshape(-1, 6 * Np)
        es = np.einsum("ki,ki->k", MS, np.linalg.solve(MC, MS[..., None])[..., 0])
        return 0.5 * float(np.sum(self.mesh.J * (ev + es)))

    def energy_rate(self, Q: np.ndarray) -> float:
        """Semi-discrete dE/dt = sum_k J_k sum_fields q^T M r (pre-WADG brackets of Eq. ewadg)."""
        Mh = ops.mass(self.N)
        rv, rs = self.rhs_pre_wadg(Q)
        e = np.einsum("kan,nm,kam->k", Q[:, 0:3], Mh, rv) + np.einsum("ksn,nm,ksm->k", Q[:, 3:9], Mh, rs)
        return float(np.sum(self.mesh.J * e))

    def l2_error(self, Q: np.ndarray, exact, t: float, field: int = 0, q: int | None = None) -> float:
        """||q_h - q||_{L2(Omega)} of one field, rule exact to degree >= 2N+2."""
        q = q if q is not None else self.N + 3
        lam, w = ops.volume_rule(q)
        V = bb.eval_basis(self.N, lam)
        pts = np.einsum("qv,kvd->kqd", lam, self.mesh.X)
        ex = exact(pts[..., 0], pts[..., 1], pts[..., 2], t)[field]
        err = Q[:, field] @ V.T - ex
        return float(np.sqrt(np.sum(self.mesh.volume[:, None] * w[None, :] * err * err)))
