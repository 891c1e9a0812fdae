"""GPU parity of the layout-dependent engine paths that the default test configs do not reach.

* The row-layout tick SpMV (8 lanes per node row reading one mode's strided column of P) is what
  every solve with n >= 25 M DOFs runs -- i.e. all of BASELINE config 5 -- in both variants: one
  CTA per row block, and the TMA-staged persistent kernel (``stream_spmv``).  It is forced here on the
  small instances (``ss_krylov_set_option(k, "row_spmv", 1)``) and checked against the reference:
  fixed-budget history and iterate (c1, tests/golden/c1.npz) and converged fields at 1e-10
  (pipe3d, the config-5 generator's small instance; tests/golden/pipe3d.npz, small3d.npz).
* The device-side conditional-WHILE graph loop (``device_loop``) and the host-polled loop give
  bitwise-identical results.
* Concurrent ``gmres_solve`` calls on systems of one mesh (the reference's solve_modes thread pool,
  spectral.py:300-305) serialise on the operator's workspace and equal the sequential results.
"""

from concurrent.futures import ThreadPoolExecutor
from contextlib import contextmanager

import numpy as np
import pytest

from golden_util import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import FluidProps, SolverSettings, assemble_mode_system, solve_mode_systems  # noqa: E402
from paper_2009_06725_b200.assembly import get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import gmres_solve  # noqa: E402
from paper_2009_06725_b200.workloads import C1_TOL, c1_case, c5_small, pipe3d_case  # noqa: E402


@contextmanager
def workspace_option(op, restart, nb, hist_cap, name, value):
    """Create (or reuse) the operator's cached workspace and set a native option for the block."""
    ws = op.krylov(restart, nb, hist_cap)
    before = ws.options()[name]
    ws.set_option(name, value)
    assert ws.options()[name] == value
    try:
        yield ws
    finally:
        ws.set_option(name, before)


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_row_layout_fixed_budget_matches_reference():
    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    g = golden("c1.npz")
    s = assemble_mode_system(case.qmesh, props, case.omegas[1], h_mode=case.h_modes()[1])
    with workspace_option(s.operator, 200, 1, 200, "row_spmv", 1):
        x, rep = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=200, max_iterations=200))
    assert rep.iterations == 200
    np.testing.assert_allclose(rep.residual_history, g["budget_hist"], rtol=1e-6)
    assert _rel(x, g["budget_x"]) <= 1e-8
    # and the same workspace back on the interleaved kernel agrees with it
    x2, rep2 = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=200, max_iterations=200))
    np.testing.assert_allclose(rep2.residual_history, rep.residual_history, rtol=1e-9)


@pytest.mark.parametrize("staged", [0, 1])
@pytest.mark.parametrize("which", ["pipe3d", "c5_small"])
def test_row_layout_converged_fields_match_reference(which, staged):
    if which == "pipe3d":
        case, g, idx = pipe3d_case(), golden("pipe3d.npz"), [1, 16]
        key = lambda i, f: f"{f}_{i}"  # noqa: E731
    else:
        case, g, idx = c5_small(), golden("small3d.npz"), [1, 16]
        key = lambda i, f: f"c5_{i}_{f}"  # noqa: E731
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(case.qmesh, props)
    settings = SolverSettings(tolerance=C1_TOL, restart=200)
    with workspace_option(op, 200, len(idx), settings.max_iterations, "row_spmv", 1), \
            workspace_option(op, 200, len(idx), settings.max_iterations, "stream_spmv", staged):
        sols = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx],
                                  [case.coefficients[i] * case.profile for i in idx], None, settings)
    for s in sols:
        assert s.report.converged and s.report.residual <= C1_TOL
        assert _rel(s.velocity, g[key(s.index, "u")]) <= 1e-7
        assert _rel(s.pressure, g[key(s.index, "p")]) <= 1e-7


def test_device_loop_bitwise_equals_host_loop():
    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    idx = [2, 5]
    settings = SolverSettings(tolerance=1e-8, restart=50, max_iterations=3000)
    h = case.h_modes()
    ref = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx], None, [h[i] for i in idx], settings)
    op = get_operator(case.qmesh, props)
    with workspace_option(op, 50, len(idx), settings.max_iterations, "device_loop", 1):
        dev = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx], None, [h[i] for i in idx], settings)
    for a, b in zip(ref, dev):
        assert a.report.iterations == b.report.iterations
        assert np.array_equal(a.velocity, b.velocity) and np.array_equal(a.pressure, b.pressure)


def test_concurrent_gmres_solve_equals_sequential():
    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    settings = SolverSettings(tolerance=1e-8, restart=40, max_iterations=2000)
    systems = [assemble_mode_system(case.qmesh, props, case.omegas[i], h_mode=case.h_modes()[i]) for i in (1, 3, 6, 8)]
    seq = [gmres_solve(s, settings) for s in systems]
    with ThreadPoolExecutor(max_workers=4) as pool:
        par = list(pool.map(lambda s: gmres_solve(s, settings), systems))
    for (xa, ra), (xb, rb) in zip(seq, par):
        assert np.array_equal(xa, xb)
        assert ra.iterations == rb.iterations and ra.residual == rb.residual


@pytest.mark.parametrize("which", ["c1", "pipe3d", "c1_wide"])
def test_fused_tick_bitwise_equals_kernel_tick(which):
    """The persistent fused tick (one cooperative launch per ticks_per_graph ticks, grid barriers
    between the SpMV / A / B / C phases) makes the same sums in the same order as the four-kernel
    graphed tick: iterations, histories and solutions are bitwise equal (and converged fields match
    the reference)."""
    if which == "pipe3d":
        case, idx, restart, maxiter = pipe3d_case(), [1, 16], 200, 200_000
    else:
        case, idx = c1_case(), [1, 4, 7]
        restart, maxiter = (200, 200_000) if which == "c1" else (300, 700)
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(case.qmesh, props)
    settings = SolverSettings(tolerance=C1_TOL, restart=restart, max_iterations=maxiter)
    g = None if case.kind != "dirichlet" else [case.coefficients[i] * case.profile for i in idx]
    h = None if case.kind != "neumann" else [case.h_modes()[i] for i in idx]
    runs = {}
    for fused in (0, 1):
        with workspace_option(op, restart, len(idx), maxiter, "fused", fused) as ws:
            runs[fused] = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx], g, h, settings)
            if fused:
                assert ws.options()["fused_active"] == 1
    for a, b in zip(runs[0], runs[1]):
        assert a.report.iterations == b.report.iterations
        assert a.report.residual_history == b.report.residual_history
        assert np.array_equal(a.velocity, b.velocity) and np.array_equal(a.pressure, b.pressure)
    if which == "pipe3d":
        ref = golden("pipe3d.npz")
        for s in runs[1]:
            assert s.report.converged
            assert _rel(s.velocity, ref[f"u_{s.index}"]) <= 1e-7


def test_alternating_pass_direction_fixed_budget_matches_reference():
    """Option "pass_alt" (basis passes stream their segments forward / backward by the parity of k,
    for L2 reuse between consecutive passes) changes only the order of the passes' row sums: the
    fixed-budget history and iterate still match the reference (c1, tests/golden/c1.npz)."""
    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    g = golden("c1.npz")
    s = assemble_mode_system(case.qmesh, props, case.omegas[1], h_mode=case.h_modes()[1])
    with workspace_option(s.operator, 200, 1, 200, "pass_alt", 1):
        x, rep = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=200, max_iterations=200))
    assert rep.iterations == 200
    np.testing.assert_allclose(rep.residual_history, g["budget_hist"], rtol=1e-6)
    assert _rel(x, g["budget_x"]) <= 1e-8


def test_alternating_pass_direction_converged_batch_invariant_and_fused():
    """pass_alt on the 3D pipe: converged fields within 1e-7 of the reference, bitwise equal between
    a two-mode batch and a one-mode batch (the direction depends only on the mode's own k) and
    between the four-kernel and the persistent fused tick."""
    case, ref, idx = pipe3d_case(), golden("pipe3d.npz"), [1, 16]
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(case.qmesh, props)
    settings = SolverSettings(tolerance=C1_TOL, restart=200)
    g = [case.coefficients[i] * case.profile for i in idx]
    runs = {}
    for fused in (0, 1):
        with workspace_option(op, 200, len(idx), settings.max_iterations, "pass_alt", 1), \
                workspace_option(op, 200, len(idx), settings.max_iterations, "fused", fused):
            runs[fused] = solve_mode_systems(case.qmesh, props, idx, case.omegas[idx], g, None, settings)
    with workspace_option(op, 200, 1, settings.max_iterations, "pass_alt", 1):
        one = solve_mode_systems(case.qmesh, props, idx[1:], case.omegas[idx[1:]], g[1:], None, settings)
    for a, b in zip(runs[0], runs[1]):
        assert a.report.iterations == b.report.iterations
        assert a.report.residual_history == b.report.residual_history
        assert np.array_equal(a.velocity, b.velocity) and np.array_equal(a.pressure, b.pressure)
    assert runs[0][1].report.iterations == one[0].report.iterations
    assert np.array_equal(runs[0][1].velocity, one[0].velocity)
    for s in runs[0]:
        assert s.report.converged and s.report.residual <= C1_TOL
        assert _rel(s.velocity, ref[f"u_{s.index}"]) <= 1e-7
        assert _rel(s.pressure, ref[f"p_{s.index}"]) <= 1e-7
