"""C-ABI library: loads, exports every declared symbol, host-only helpers pinned to the paper.

CPU-only (no GPU needed): the projection / mass-inverse constants are computed by the
library's host code (closed-form eigenvalues, R8) and checked against the
values PAPER.md prints (tests/golden/), and setup fails loudly without a device.
"""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def L():
    from paper_1808_08645_b200 import lib

    return lib


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "bbwadg.h")) as fh:
        txt = fh.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(bbwadg_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(L):
    syms = _declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L._L, s), s
        assert isinstance(getattr(L._L, s), ctypes._CFuncPtr)


def test_library_is_sm100a_build(L):
    # the fatbin must carry sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "--list-elf", L.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for ln in fh:
            if ln.strip() and not ln.startswith("#"):
                rows.append([float(x) for x in ln.split()])
    return rows


def test_projection_constants_match_paper_table1(L):
    # PAPER.md Table 1, 4 printed decimals
    for row in _read_golden("table1_projection_constants.txt"):
        N, M, c = int(row[0]), int(row[1]), np.array(row[2:])
        got = L.bbwadg_projection_constants(N, M)
        assert got.shape == c.shape
        assert np.all(np.abs(got - c) <= 0.5e-4 + 1e-12), (N, M, got, c)


def test_table1_first_row_is_mislabelled():
    # the printed "N=2, M=1" row (0.6667, -0.0667) has 2 entries, so it cannot be an N=2 row
    # (c_0..c_N has N+1 entries, Thm main); R4
    from paper_1808_08645_b200 import lib as L

    assert np.allclose(L.bbwadg_projection_constants(1, 1), [2 / 3, -1 / 15], atol=1e-15)
    assert len(L.bbwadg_projection_constants(2, 1)) == 3


def test_mass_inverse_constants_match_paper_table2(L):
    # PAPER.md Table 2, exact as printed
    for row in _read_golden("table2_mass_inverse_constants.txt"):
        N, c = int(row[0]), np.array(row[1:])
        got = L.bbwadg_mass_inverse_constants(N)
        assert np.allclose(got, c, rtol=1e-12, atol=1e-9), (N, got, c)


def test_condition_numbers_match_section_4_4(L):
    # sum |c_j| ~ 1.67e7 for M^-1 (N=7), ~14.53 (M=1) and ~41.35 (M=2) for P^{N+M}_N (N=7)
    assert abs(np.abs(L.bbwadg_mass_inverse_constants(7)).sum() / 1.67e7 - 1) < 0.01
    assert abs(np.abs(L.bbwadg_projection_constants(7, 1)).sum() - 14.53) < 0.01
    assert abs(np.abs(L.bbwadg_projection_constants(7, 2)).sum() - 41.35) < 0.01


def test_projection_constants_reproduce_projection_identity(L):
    # P^{N+M}_N applied to an elevated degree-N polynomial returns it (projection is the
    # identity on P^N): sum_j c_j lambda^{N-j}_k = lambda^{N+M}_k with k = N (modal degree N)
    # reduces to c_0 = lambda^{N+M}_N / lambda^N_N; check against the closed form ratio.
    from math import factorial

    def lam(n, k):
        return factorial(n) ** 2 * 6 / (factorial(n + k + 3) * factorial(n - k))

    for N, M in [(2, 1), (5, 3), (7, 4), (9, 9)]:
        c0 = L.bbwadg_projection_constants(N, M)[0]
        assert abs(c0 - lam(N + M, N) / lam(N, N)) < 1e-13 * abs(c0)


def test_setup_without_device_fails_loudly(L):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from workloads import kuhn

    v, e = kuhn.kuhn_mesh(1)
    with pytest.raises(L.BBWADGError, match="NO_DEVICE"):
        L.bbwadg_setup(v, e, 3, 1, np.ones((len(e), 4)), L.bbwadg_default_options())


def test_setup_validates_arguments_before_device(L):
    # host-side validation runs before the device query, so these fail with their own status even
    # on a machine without a GPU (status names, not just "an error")
    v = np.zeros((4, 3))
    e = np.array([[0, 1, 2, 3]], dtype=np.int64)
    with pytest.raises(L.BBWADGError, match="MESH"):  # degenerate tet: J = 0
        L.bbwadg_setup(v, e, 3, 1, np.ones((1, 4)), L.bbwadg_default_options())
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    with pytest.raises(L.BBWADGError, match="UNSUPPORTED"):  # N > 9
        L.bbwadg_setup(v, e, 10, 1, np.ones((1, 4)), L.bbwadg_default_options())
    with pytest.raises(L.BBWADGError, match="UNSUPPORTED"):  # M > N
        L.bbwadg_setup(v, e, 2, 3, np.ones((1, 20)), L.bbwadg_default_options())


def test_elastic_and_2d_setups_validate_before_device(L):
    # bbwadg_elastic_setup / bbwadg2d_setup check arguments and the mesh on the host before any device call
    from workloads import kuhn, tri2d

    v, e = kuhn.kuhn_mesh(1)
    K = len(e)
    ones = np.ones((K, 4))
    o = L.bbwadg_default_options()
    o.world_size, o.rank = 2, 0
    with pytest.raises(L.BBWADGError, match="UNSUPPORTED"):  # elastic contexts are single-GPU
        L.bbwadg_elastic_setup(v, e, 3, 1, ones, ones, ones, o)
    with pytest.raises(L.BBWADGError, match="UNSUPPORTED"):  # N > 9
        L.bbwadg_elastic_setup(v, e, 10, 1, ones, ones, ones, L.bbwadg_default_options())
    v2, e2 = tri2d.tri_mesh(2)
    c2 = np.ones((len(e2), 3))
    with pytest.raises(L.BBWADGError, match="MESH"):  # clockwise triangles are rejected, never reordered
        L.bbwadg2d_setup(v2, np.ascontiguousarray(e2[:, [0, 2, 1]]), 3, 1, c2, L.bbwadg_default_options())
    with pytest.raises(L.BBWADGError, match="NONPOSITIVE_C2"):
        L.bbwadg2d_setup(v2, e2, 3, 1, -c2, L.bbwadg_default_options())
    with pytest.raises(L.BBWADGError, match="UNSUPPORTED"):  # M > N
        L.bbwadg2d_setup(v2, e2, 2, 3, np.ones((len(e2), 10)), L.bbwadg_default_options())
    bad = np.ascontiguousarray(e2.copy())
    bad[0, 0] = 10 ** 6
    with pytest.raises(L.BBWADGError, match="MESH"):  # vertex id out of range
        L.bbwadg2d_setup(v2, bad, 3, 1, c2, L.bbwadg_default_options())
    o = L.bbwadg_default_options()
    o.halo_transport = 2
    with pytest.raises(L.BBWADGError, match="INVALID_ARG"):
        L.bbwadg_setup(v, e, 3, 1, ones, o)
