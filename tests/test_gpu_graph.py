"""bbwadg_run replays one LSRK step as a CUDA graph (single-partition contexts without a source): the
result must be bitwise equal to stepping with individual launches (bbwadg_step), for every kernel family,
across runs that start from either ping-pong buffer and after a dt change (graph rebuild)."""
import os

import numpy as np
import pytest

from workloads import elastic as ew
from workloads import kuhn, media, states, tri2d

pytestmark = pytest.mark.gpu


def _make(kind, N, M):
    from paper_1808_08645_b200 import ElasticSolver, Solver, Solver2D

    if kind == "acoustic":
        v, e = kuhn.kuhn_mesh(3)
        return Solver(v, e, N, M, media.random_c2(len(e), M)), states.random_state(len(e), N)
    if kind == "elastic":
        v, e = kuhn.kuhn_mesh(2)
        return ElasticSolver(v, e, N, M, *ew.random_material(len(e), M)), ew.random_state(len(e), N)
    v, e = tri2d.tri_mesh(6)
    return Solver2D(v, e, N, M, tri2d.random_c2(len(e), M)), tri2d.random_state(len(e), N)


@pytest.mark.parametrize("kind,N,M", [("acoustic", 3, 1), ("acoustic", 7, 4), ("acoustic", 2, 2),
                                      ("elastic", 3, 1), ("2d", 4, 2)])
def test_graph_run_is_bitwise_equal_to_steps(gpu_lib, kind, N, M):
    s, Q0 = _make(kind, N, M)
    dt = 1e-3
    s.set_state(Q0)
    s.run(0.0, dt, 3)          # graph (3 steps: starts on buffer 0)
    s.run(3 * dt, dt, 2)       # graph, starting from the other buffer
    s.run(5 * dt, 0.5 * dt, 2)  # dt change: graphs rebuilt
    a = s.get_state()
    s.set_state(Q0)
    for i in range(3):
        s.step(i * dt, dt)
    for i in range(2):
        s.step((3 + i) * dt, dt)
    for i in range(2):
        s.step(5 * dt + i * 0.5 * dt, 0.5 * dt)
    b = s.get_state()
    assert np.array_equal(a, b)
    os.environ["BBWADG_NO_GRAPH"] = "1"
    try:
        s.set_state(Q0)
        s.run(0.0, dt, 3)
        s.run(3 * dt, dt, 2)
        s.run(5 * dt, 0.5 * dt, 2)
        assert np.array_equal(s.get_state(), a)
    finally:
        del os.environ["BBWADG_NO_GRAPH"]
