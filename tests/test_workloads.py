"""Input generators: Kuhn meshes, media, states (shapes, structure, invariants)."""
import numpy as np
import pytest

from workloads import kuhn, media, states


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_kuhn_mesh_volume_orientation_conformity(n):
    v, e = kuhn.kuhn_mesh(n)
    assert e.shape == (6 * n ** 3, 4)
    X = v[e]
    det = np.einsum("ki,ki->k", X[:, 1] - X[:, 0], np.cross(X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]))
    assert np.all(det > 0)
    assert abs(det.sum() / 6 - 8.0) < 1e-12
    # every face is shared by <= 2 elements; boundary faces = 2 per cube face on the surface
    faces = np.sort(np.concatenate([e[:, [1, 2, 3]], e[:, [0, 2, 3]], e[:, [0, 1, 3]], e[:, [0, 1, 2]]]), axis=1)
    _, counts = np.unique(faces, axis=0, return_counts=True)
    assert counts.max() == 2
    assert (counts == 1).sum() == 6 * n * n * 2


def test_kuhn_box_and_morton_locality():
    v, e = kuhn.kuhn_mesh((4, 2, 2), h=0.5)
    assert e.shape[0] == 6 * 16
    c = v[e].mean(1)
    # consecutive cubes (6 tets each) are Morton neighbours: centroid steps stay small on average
    cc = c.reshape(-1, 6, 3).mean(1)
    assert np.mean(np.linalg.norm(np.diff(cc, axis=0), axis=1)) < 1.0


def test_config_sizes():
    # BASELINE.json configs: 48, 384/3072/24576, 511104, 1053696, 4088832 tets
    for n, K in [(2, 48), (4, 384), (8, 3072), (16, 24576), (44, 511104), (56, 1053696), (88, 4088832)]:
        assert 6 * n ** 3 == K


def test_media_projection_recovers_polynomials():
    v, e = kuhn.kuhn_mesh(2)
    M = 2
    f = lambda x, y, z: 1.0 + 0.1 * x * y - 0.2 * z * z  # noqa: E731  in P^2
    c = media.project_c2(v, e, f, M)
    # evaluate at vertices: Bernstein vertex coefficients are vertex values
    from math import comb
    assert c.shape == (len(e), comb(M + 3, 3))
    X = v[e]
    # vertex 1 <-> multi-index (0, M, 0, 0) at canonical position M
    assert np.allclose(c[:, M], f(*X[:, 1].T), atol=1e-12)


def test_layered_media_positive_at_config4_degree():
    v, e = kuhn.kuhn_mesh(8)
    c = media.project_c2(v, e, media.c2_layered(), 3)
    assert media.min_value(c, 3, 8) > 0.25


def test_random_inputs_seeded():
    a = states.random_state(5, 3)
    b = states.random_state(5, 3)
    assert np.array_equal(a, b) and a.shape == (5, 4, 20)
    c = media.random_c2(5, 2)
    assert c.min() >= 0.5 and c.max() <= 1.5 and c.shape == (5, 10)
