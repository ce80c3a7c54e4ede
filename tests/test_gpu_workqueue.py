"""The stage kernels take element batches from a per-context global work queue (DESIGN.md §6 "Work queue").
Every element's stage is independent of which warp computes it and when, so the result must be BITWISE the
same whatever the schedule: the default persistent grid (each unit draws about one ticket on these meshes)
against a grid of one CTA per SM (BBWADG_BLOCKS_PER_SM=1: every unit draws several tickets, and the
last-unit counter reset is exercised on every launch).  A skipped or duplicated batch, or a counter left
non-zero for the next launch, breaks the equality (or the finiteness of the state)."""
import os

import numpy as np
import pytest
import torch

from workloads import elastic as ew
from workloads import kuhn, media, states

pytestmark = pytest.mark.gpu


def _acoustic(N, M, n, dtype, blocks):
    from paper_1808_08645_b200 import Solver

    old = os.environ.get("BBWADG_BLOCKS_PER_SM")
    if blocks:
        os.environ["BBWADG_BLOCKS_PER_SM"] = str(blocks)
    try:
        v, e = kuhn.kuhn_mesh(n)
        s = Solver(v, e, N, M, media.random_c2(len(e), M), dtype=dtype)
    finally:
        if old is None:
            os.environ.pop("BBWADG_BLOCKS_PER_SM", None)
        else:
            os.environ["BBWADG_BLOCKS_PER_SM"] = old
    return s, len(e)


@pytest.mark.parametrize("N,M,n,dtype", [(3, 1, 6, "f64"), (7, 4, 6, "f64"), (9, 9, 4, "f64"), (5, 3, 6, "f32"),
                                         (2, 2, 8, "f64")])
def test_schedule_independent_bitwise(gpu_lib, N, M, n, dtype):
    Q0 = None
    outs = []
    for blocks in (0, 1):
        s, K = _acoustic(N, M, n, dtype, blocks)
        if Q0 is None:
            Q0 = states.random_state(K, N)
        td = torch.float64 if dtype == "f64" else torch.float32
        r = s.rhs(torch.tensor(Q0, dtype=td, device="cuda"), 0.25).cpu().numpy()
        s.set_state(Q0)
        s.run(0.0, 1e-3, 4)  # 20 stage launches: each must start from a reset queue
        for i in range(3):
            s.step((4 + i) * 1e-3, 1e-3)
        q = s.get_state()
        info = s.info()
        s.close()
        assert np.all(np.isfinite(q))
        outs.append((r, q, info))
    (r0, q0, i0), (r1, q1, i1) = outs
    assert np.array_equal(r0, r1)
    assert np.array_equal(q0, q1)


def test_two_contexts_interleaved(gpu_lib):
    """Two contexts own separate queues: interleaving their launches on the default stream gives the same
    states as running each alone."""
    from paper_1808_08645_b200 import Solver

    v, e = kuhn.kuhn_mesh(6)
    a = Solver(v, e, 7, 4, media.random_c2(len(e), 4))
    b = Solver(v, e, 5, 2, media.random_c2(len(e), 2, lo=0.8, hi=1.2))
    Qa, Qb = states.random_state(len(e), 7), states.random_state(len(e), 5)
    a.set_state(Qa)
    b.set_state(Qb)
    for i in range(5):
        a.step(i * 1e-3, 1e-3)
        b.step(i * 1e-3, 1e-3)
    qa, qb = a.get_state(), b.get_state()
    a.set_state(Qa)
    a.run(0.0, 1e-3, 5)
    b.set_state(Qb)
    b.run(0.0, 1e-3, 5)
    assert np.array_equal(a.get_state(), qa)
    assert np.array_equal(b.get_state(), qb)


def test_elastic_schedule_independent_bitwise(gpu_lib):
    from paper_1808_08645_b200 import ElasticSolver

    v, e = kuhn.kuhn_mesh(4)
    mat = ew.random_material(len(e), 2)
    Q0 = ew.random_state(len(e), 7)
    outs = []
    for blocks in (0, 1):
        old = os.environ.get("BBWADG_BLOCKS_PER_SM")
        if blocks:
            os.environ["BBWADG_BLOCKS_PER_SM"] = "1"
        try:
            s = ElasticSolver(v, e, 7, 2, *mat)
        finally:
            if old is None:
                os.environ.pop("BBWADG_BLOCKS_PER_SM", None)
        s.set_state(Q0)
        s.run(0.0, 1e-3, 3)
        outs.append(s.get_state())
        s.close()
    assert np.array_equal(outs[0], outs[1])
