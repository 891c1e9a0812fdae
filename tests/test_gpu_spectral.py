"""GPU end-to-end parity: solve_modes + reconstruct against the reference's converged fields.

Bar (BASELINE.json north_star): modal velocity/pressure within relative L2 1e-7 of the reference
when both are converged to relative residual 1e-10.
"""

import numpy as np
import pytest

import oracle
from golden_util import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import (  # noqa: E402
    BoundaryWaveform, FluidProps, SolverSettings, fourier_transform_bcs, reconstruct, reconstruct_series,
    solve_mode_systems, solve_modes,
)
from paper_2009_06725_b200.workloads import C1_TOL, c1_case, pipe3d_case  # noqa: E402

SETTINGS = SolverSettings(tolerance=1e-9)


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(scope="module")
def c1_solution():
    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    wf = BoundaryWaveform(patch="inlet", kind="neumann", direction=np.array([1.0, 0.0]), period=case.period,
                          coefficients=case.coefficients)
    ms = fourier_transform_bcs([wf], case.n_modes)
    sols = solve_modes(case.qmesh, props, ms, SolverSettings(tolerance=C1_TOL, restart=200))
    return case, sols, golden("c1.npz")


def test_c1_all_modes_match_reference(c1_solution):
    case, sols, g = c1_solution
    for i, s in enumerate(sols):
        assert s.index == i and s.report.converged and s.report.residual <= C1_TOL
        assert _rel(s.velocity, g[f"u_{i}"]) <= 1e-7, i
        assert _rel(s.pressure, g[f"p_{i}"]) <= 1e-7, i
        # iteration counts within a few percent of the reference's (rounding-order differences only)
        ref_it = int(g[f"iters_{i}"])
        assert abs(s.report.iterations - ref_it) <= max(50, 0.05 * ref_it)


def test_c1_reconstruct_32_samples(c1_solution):
    case, sols, g = c1_solution
    ts = np.arange(32) / 32.0
    U, P = reconstruct_series(sols, ts)
    vel = [s.velocity for s in sols]
    pre = [s.pressure for s in sols]
    for j, t in enumerate(ts):
        u, p = oracle.reconstruct(vel, pre, [s.omega for s in sols], float(t))
        assert np.array_equal(U[j], u) or np.abs(U[j] - u).max() <= 1e-15 * max(1.0, np.abs(u).max())
        assert np.abs(P[j] - p).max() <= 1e-15 * max(1.0, np.abs(p).max())
    for j, t in enumerate(g["recon_t"]):
        u, p = reconstruct(sols, float(t))
        assert _rel(u, g[f"recon_u_{j}"]) <= 1e-7 and _rel(p, g[f"recon_p_{j}"]) <= 1e-7


def test_reconstruct_bitwise_against_oracle_on_reference_fields():
    g = golden("c1.npz")
    from paper_2009_06725_b200.krylov import SolveReport
    from paper_2009_06725_b200.spectral import ModeSolution

    sols = [ModeSolution(i, float(g["omegas"][i]), g[f"u_{i}"], g[f"p_{i}"], SolveReport(0, 0.0, True, 0.0))
            for i in range(9)]
    for j, t in enumerate(g["recon_t"]):
        u, p = reconstruct(sols, float(t))
        np.testing.assert_allclose(u, g[f"recon_u_{j}"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(p, g[f"recon_p_{j}"], rtol=0, atol=1e-15)


def _wave(coeffs, kind="neumann", patch="inlet"):
    return BoundaryWaveform(patch=patch, kind=kind, direction=np.array([1.0, 0.0]), period=1.0,
                            coefficients=np.asarray(coeffs, complex))


def test_zero_coefficient_mode_short_circuits(small_channel_qmesh, fluid):
    ms = fourier_transform_bcs([_wave([0.0, 1.0, 0.0])], 2)
    sols = solve_modes(small_channel_qmesh, fluid, ms, SETTINGS)
    assert sols[0].report.iterations == 0 and np.all(sols[0].velocity == 0)
    assert sols[2].report.iterations == 0 and sols[1].report.iterations > 0


def test_amplitude_threshold_selects_nonconsecutive_modes(small_channel_qmesh, fluid):
    ms = fourier_transform_bcs([_wave([0.0, 1.0, 0.01, 0.6, 0.005])], 4).thresholded(0.1)
    sols = solve_modes(small_channel_qmesh, fluid, ms, SETTINGS)
    assert [s.index for s in sols if s.report.iterations > 0] == [1, 3]


def test_reconstruct_phases(small_channel_qmesh, fluid):
    sols = solve_modes(small_channel_qmesh, fluid, fourier_transform_bcs([_wave([0.0, 1.0])], 1), SETTINGS)
    u0, _ = reconstruct(sols, 0.0)
    uq, _ = reconstruct(sols, 0.25)
    assert np.allclose(u0, sols[1].velocity.real, atol=1e-14)
    assert np.allclose(uq, -sols[1].velocity.imag, atol=1e-12)


def test_reconstruct_steady_time_independent(small_channel_qmesh, fluid):
    sols = solve_modes(small_channel_qmesh, fluid, fourier_transform_bcs([_wave([1.0])], 0), SETTINGS)
    ua, _ = reconstruct(sols, 0.123)
    ub, _ = reconstruct(sols, 0.789)
    assert np.array_equal(ua, ub)
    assert np.abs(sols[0].velocity.imag).max() < 1e-12


def test_reconstruct_two_modes_matches_bruteforce(small_channel_qmesh, fluid):
    sols = solve_modes(small_channel_qmesh, fluid, fourier_transform_bcs([_wave([0.3, 1.0, 0.2 - 0.4j])], 2), SETTINGS)
    ts = np.random.default_rng(1).uniform(0.0, 1.0, 100)
    U, _ = reconstruct_series(sols, ts)
    for j, t in enumerate(ts):
        ref = sum(np.real(s.velocity * np.exp(1j * s.omega * t)) for s in sols)
        assert np.allclose(U[j], ref, atol=1e-15)


def test_mode_order_and_batch_bitwise(small_channel_qmesh, fluid):
    ms = fourier_transform_bcs([_wave([0.5, 1.0, 0.3 + 0.2j])], 2)
    a = solve_modes(small_channel_qmesh, fluid, ms, SETTINGS, workers=1)
    b = solve_modes(small_channel_qmesh, fluid, ms, SETTINGS, workers=3)
    perm = type(ms)(indices=ms.indices[::-1], frequencies=ms.frequencies, period=ms.period,
                    coefficients=ms.coefficients, waveforms=ms.waveforms)
    c = solve_modes(small_channel_qmesh, fluid, perm, SETTINGS)[::-1]
    for x, y, z in zip(a, b, c):
        assert np.array_equal(x.velocity, y.velocity) and np.array_equal(x.pressure, y.pressure)
        assert np.array_equal(x.velocity, z.velocity)


def test_linearity_in_boundary_data(small_channel_qmesh, fluid):
    alpha = 0.7 - 1.3j
    ms = fourier_transform_bcs([_wave([0.2, 1.0])], 1)
    base = solve_modes(small_channel_qmesh, fluid, ms, SETTINGS)
    scaled = solve_modes(small_channel_qmesh, fluid, ms.scaled(alpha), SETTINGS)
    for a, b in zip(base, scaled):
        ref = np.linalg.norm(alpha * a.velocity)
        assert np.linalg.norm(b.velocity - alpha * a.velocity) / ref < 10 * SETTINGS.tolerance


def test_pipe3d_modes_match_reference():
    """Down-scaled 3D pipe, parabolic Dirichlet inlet: modes 1 and 16 converged to 1e-10."""
    case = pipe3d_case()
    g = golden("pipe3d.npz")
    props = FluidProps(case.density, case.viscosity)
    idx = [1, 16]
    sols = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx], [case.coefficients[i] * case.profile for i in idx],
                              None, SolverSettings(tolerance=C1_TOL, restart=200))
    for s in sols:
        assert s.report.converged and s.report.residual <= C1_TOL
        assert _rel(s.velocity, g[f"u_{s.index}"]) <= 1e-7
        assert _rel(s.pressure, g[f"p_{s.index}"]) <= 1e-7
