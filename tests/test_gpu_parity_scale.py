"""LSRK-stage parity (bbwadg_step, mode 0) on meshes large enough that every persistent CTA
group runs its grid-stride batch loop more than once, with per-field / per-element maxima next
to the pooled relative L2 error, plus GPU energy stability and time-dependent-source stage times.

Bars (BASELINE.json north_star): fp64 <= 1e-10 after many steps (<= 1e-11 after 2), fp32 <= 1e-5.
Meshes: Kuhn n = 8 (3,072 tets) for N >= 5 (grid = 148 SMs x 4 CTAs x 4 whole-warp groups = 2,368
element slots for TG = 32, 1,184 for TG = 64), n = 16 (24,576 tets) for sub-warp groups (N <= 4:
up to 32 elements per CTA).  Inputs: seeded random states (rng 1808) and c^2 (rng 808).
"""
import numpy as np
import pytest

from oracle.acoustic import AcousticOracle
from workloads import kuhn, media, states

pytestmark = pytest.mark.gpu


def errors(out, ref):
    """(pooled relative L2, max over fields c and elements k of ||out-ref||_inf(k,c) / ||ref||_inf(:,c))."""
    rel = float(np.linalg.norm((out - ref).ravel()) / np.linalg.norm(ref.ravel()))
    scale = np.max(np.abs(ref), axis=(0, 2))  # per field
    per = np.max(np.abs(out - ref), axis=2) / scale[None, :]  # [K, 4]
    return rel, float(per.max()), np.unravel_index(int(np.argmax(per)), per.shape)


def _run_both(N, M, n, nsteps, dtype="f64", source=False):
    from paper_1808_08645_b200 import Solver

    v, e = kuhn.kuhn_mesh(n)
    c2 = media.random_c2(len(e), M)
    Q0 = states.random_state(len(e), N)
    dt = 0.5 * kuhn.min_height(v, e) / (np.sqrt(1.5) * (N + 1) ** 2)
    g = None
    if source:
        g = 50.0 * np.random.default_rng(11).standard_normal((len(e), states.num_coeffs(N)))
    o = AcousticOracle(v, e, N, M, c2, source=g)
    s = Solver(v, e, N, M, c2, dtype=dtype)
    if g is not None:
        s.set_source(g)
    t0 = 0.3 if source else 0.0
    s.set_state(Q0)
    s.run(t0, dt, nsteps)
    out = s.get_state().astype(np.float64)
    ref = o.run(Q0, t0, dt, nsteps)
    s.close()
    return out, ref


@pytest.mark.parametrize("N,M,n", [(7, 4, 8), (9, 9, 8), (2, 2, 16), (5, 3, 8)])
def test_lsrk_stage_parity_grid_stride(gpu_lib, N, M, n):
    out, ref = _run_both(N, M, n, 2)
    rel, mx, where = errors(out, ref)
    assert rel <= 1e-11 and mx <= 1e-10, (rel, mx, where)


def test_lsrk_stage_parity_fp32_grid_stride(gpu_lib):
    out, ref = _run_both(5, 3, 8, 2, dtype="f32")
    rel, mx, where = errors(out, ref)
    assert rel <= 1e-5 and mx <= 1e-4, (rel, mx, where)


def test_20_steps_config5_degree(gpu_lib):
    # BASELINE config 5's (N, M) = (7, 4), 20 LSRK45 steps on a mesh that iterates the batch loop
    out, ref = _run_both(7, 4, 8, 20)
    rel, mx, where = errors(out, ref)
    assert rel <= 1e-10 and mx <= 1e-9, (rel, mx, where)


def test_time_dependent_source_stage_times(gpu_lib):
    # a large source g sin(pi t) makes every stage time c_s dt visible (the GPU's RK_C is its own
    # transcription of Carpenter-Kennedy; a 1e-6 error in one c_s moves the result by >> 1e-10)
    out, ref = _run_both(3, 2, 4, 10, source=True)
    rel, mx, where = errors(out, ref)
    assert rel <= 1e-10 and mx <= 1e-9, (rel, mx, where)


def test_energy_non_increasing_on_gpu(gpu_lib):
    # P:136-137 (energy stability with tau >= 0, R22): the WADG energy of the GPU states
    # never increases over LSRK steps
    from paper_1808_08645_b200 import Solver

    N, M = 4, 2
    v, e = kuhn.kuhn_mesh(4)
    c2 = media.random_c2(len(e), M)
    o = AcousticOracle(v, e, N, M, c2)
    s = Solver(v, e, N, M, c2)
    s.set_state(states.random_state(len(e), N))
    dt = 0.5 * kuhn.min_height(v, e) / (np.sqrt(1.5) * (N + 1) ** 2)
    E0 = o.energy(s.get_state())
    for it in range(10):
        s.run(it * dt, dt, 1)
        E1 = o.energy(s.get_state())
        assert E1 <= E0 * (1 + 1e-13), (it, E0, E1)
        E0 = E1
    s.close()
