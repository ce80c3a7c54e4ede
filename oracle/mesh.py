"""Geometry and connectivity of an affine tetrahedral mesh (oracle's own).

Each element D^k is the affine image of D^:
    x = X0 + sum_{i=1..3} l_i (X_i - X0),   l_i = (1 + r_i)/2,
so dx/d(r,s,t) = [X1-X0, X2-X0, X3-X0] / 2, J^k = det(dx/dr) = |T_k|/|D^|,
and G^k = (dx/dr)^-1 holds the geometric factors r_x, s_x, ....
Face f is the face opposite local vertex f; its outward unit normal points away
from vertex f.  Neighbours are found by matching the sorted global vertex
triple of each face (conforming meshes: at most two elements per face).

For the surface term the oracle needs, for every element face, the
barycentric coordinates *in the neighbour* of the physical face quadrature
points of this element: they are obtained by inverting the neighbour's affine
map at those physical points (no face-orientation tables).
"""
from __future__ import annotations

import numpy as np

from . import bernstein as bb
from . import operators as ops


class OracleMesh:
    def __init__(self, vertices: np.ndarray, elements: np.ndarray):
        self.vertices = np.asarray(vertices, dtype=np.float64)
        self.elements = np.asarray(elements, dtype=np.int64)
        X = self.vertices[self.elements]  # K,4,3
        self.X = X
        K = X.shape[0]
        self.K = K
        E = np.stack([X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]], axis=-1)  # K,3(x),3(i)
        self.dxdr = E / 2.0
        self.J = np.linalg.det(self.dxdr)
        if np.any(self.J <= 0):
            raise ValueError("element with non-positive Jacobian")
        self.G = np.linalg.inv(self.dxdr)  # G[k, ref, phys] = d r_ref / d x_phys
        self.Einv = np.linalg.inv(E)  # l_{1..3} = Einv (x - X0)
        self.volume = self.J * float(bb.REF_VOLUME)
        # faces
        self.area = np.zeros((K, 4))
        self.normal = np.zeros((K, 4, 3))
        keys = np.zeros((K, 4, 3), dtype=np.int64)
        for f in range(4):
            o = [v for v in range(4) if v != f]
            c = np.cross(X[:, o[1]] - X[:, o[0]], X[:, o[2]] - X[:, o[0]])
            a2 = np.linalg.norm(c, axis=1)
            n = c / a2[:, None]
            sgn = np.sign(np.einsum("kd,kd->k", n, X[:, o[0]] - X[:, f]))
            self.normal[:, f] = n * sgn[:, None]
            self.area[:, f] = 0.5 * a2
            keys[:, f] = np.sort(self.elements[:, o], axis=1)
        # neighbour matching through sorted vertex triples
        flat = keys.reshape(-1, 3)
        order = np.lexsort((flat[:, 2], flat[:, 1], flat[:, 0]))
        sk = flat[order]
        same = np.all(sk[1:] == sk[:-1], axis=1)
        if np.any(same[1:] & same[:-1]):
            raise ValueError("face shared by more than two elements")
        self.nbr = -np.ones(K * 4, dtype=np.int64)
        a, b = order[:-1][same], order[1:][same]
        self.nbr[a] = b // 4
        self.nbr[b] = a // 4
        self.nbr = self.nbr.reshape(K, 4)
        self._nbr_lam = {}

    def face_points(self, n: int):
        """Physical face quadrature points [K,4,nq,3] of the degree-n face rule."""
        lams, _, _ = ops.face_ops(n)
        return np.stack([np.einsum("qv,kvd->kqd", lams[f], self.X) for f in range(4)], axis=1)

    def barycentric(self, k: np.ndarray, x: np.ndarray) -> np.ndarray:
        """Barycentric coordinates in element(s) k of points x[..., 3]."""
        l123 = np.einsum("kij,k...j->k...i", self.Einv[k], x - self.X[k, 0][:, None, :])
        return np.concatenate([1.0 - l123.sum(-1, keepdims=True), l123], axis=-1)

    def neighbour_trace_matrices(self, n: int) -> np.ndarray:
        """Vnb[k, f] = B^n evaluated in the neighbour at this element's face
        points, [K,4,nq,Np] (zeros on boundary faces)."""
        if n in self._nbr_lam:
            return self._nbr_lam[n]
        pts = self.face_points(n)  # K,4,nq,3
        K = self.K
        nq = pts.shape[2]
        out = np.zeros((K, 4, nq, bb.num_coeffs(n)))
        for f in range(4):
            nb = self.nbr[:, f]
            m = nb >= 0
            lam = self.barycentric(nb[m], pts[m, f])
            out[m, f] = bb.eval_basis(n, lam)
        self._nbr_lam[n] = out
        return out
