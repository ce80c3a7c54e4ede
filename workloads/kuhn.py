"""Kuhn-cube tetrahedral meshes (input data only).

The paper's convergence meshes are GMSH uniform meshes that are
not available; reading R12 the domain
[-1,1]^3 is split into n^3 cubes of side h = 2/n, each cut into the 6 Kuhn
tetrahedra that share the cube's main diagonal.  The triangulation is
conforming, every element is positively oriented
(det[X1-X0, X2-X0, X3-X0] > 0, the orientation of the reference tetrahedron of
P:56/P:66), and cubes are ordered along a Morton (Z-order) curve so that
consecutive elements are spatial neighbours (HBM/L2 locality of neighbour
traces on the GPU; contiguous element ranges are compact partitions).

Returned arrays are plain numpy: ``vertices`` float64 [nv,3] and ``elements``
int64 [K,4] (global vertex ids per element, local vertex i <-> barycentric
lambda_i).
"""
from __future__ import annotations

import itertools

import numpy as np

# The 6 permutations of the axes; the Kuhn tet for permutation pi has vertices
# 0, e_pi0, e_pi0+e_pi1, (1,1,1) (cube-local corner offsets).
_PERMS = list(itertools.permutations(range(3)))


def _perm_sign(p) -> int:
    s = 1
    p = list(p)
    for i in range(3):
        for j in range(i + 1, 3):
            if p[i] > p[j]:
                s = -s
    return s


def _morton3(i: np.ndarray, j: np.ndarray, k: np.ndarray) -> np.ndarray:
    code = np.zeros(i.shape, dtype=np.uint64)
    for b in range(21):
        code |= ((i.astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
        code |= ((j.astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + 1)
        code |= ((k.astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + 2)
    return code


def kuhn_mesh(n, h: float | None = None, origin=(-1.0, -1.0, -1.0)):
    """Kuhn mesh of an (nx, ny, nz) block of cubes.

    ``n`` is an int (n^3 cubes on [-1,1]^3, h = 2/n) or a tuple (nx, ny, nz)
    (then ``h`` defaults to 2/max(n) and the box extends from ``origin``).
    K = 6 * nx * ny * nz.
    """
    if np.isscalar(n):
        nx = ny = nz = int(n)
    else:
        nx, ny, nz = (int(v) for v in n)
    if min(nx, ny, nz) < 1:
        raise ValueError("need at least one cube per direction")
    if h is None:
        h = 2.0 / max(nx, ny, nz)
    ox, oy, oz = origin
    # vertices, lexicographic in (i, j, k)
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    vid = lambda i, j, k: i + (nx + 1) * (j + (ny + 1) * k)  # noqa: E731
    verts = np.zeros(((nx + 1) * (ny + 1) * (nz + 1), 3), dtype=np.float64)
    flat = vid(ii, jj, kk).ravel()
    verts[flat, 0] = ox + h * ii.ravel()
    verts[flat, 1] = oy + h * jj.ravel()
    verts[flat, 2] = oz + h * kk.ravel()

    # cubes in Morton order
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = ci.ravel(), cj.ravel(), ck.ravel()
    order = np.argsort(_morton3(ci, cj, ck), kind="stable")
    ci, cj, ck = ci[order], cj[order], ck[order]

    ncube = ci.size
    elems = np.zeros((ncube, 6, 4), dtype=np.int64)
    for t, p in enumerate(_PERMS):
        corners = [np.zeros(3, dtype=np.int64)]
        c = np.zeros(3, dtype=np.int64)
        for ax in p:
            c = c.copy()
            c[ax] += 1
            corners.append(c)
        ids = [vid(ci + o[0], cj + o[1], ck + o[2]) for o in corners]
        if _perm_sign(p) < 0:  # det = sign(pi); swap local vertices 2,3 to fix orientation
            ids[2], ids[3] = ids[3], ids[2]
        for lv in range(4):
            elems[:, t, lv] = ids[lv]
    return verts, elems.reshape(-1, 4)


def min_height(vertices: np.ndarray, elements: np.ndarray) -> float:
    """Smallest tetrahedron height 3|T|/|f| over all element faces (the h_min of
    the dt rule, R14)."""
    X = vertices[elements]  # K,4,3
    vol6 = np.abs(np.einsum("ki,ki->k", X[:, 1] - X[:, 0], np.cross(X[:, 2] - X[:, 0], X[:, 3] - X[:, 0])))
    hmin = np.inf
    for f in range(4):
        o = [v for v in range(4) if v != f]
        a2 = np.linalg.norm(np.cross(X[:, o[1]] - X[:, o[0]], X[:, o[2]] - X[:, o[0]]), axis=1)
        hmin = min(hmin, float(np.min(vol6 / a2)))
    return hmin
