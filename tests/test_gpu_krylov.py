"""GPU GMRES contracts: the reference's own krylov tests (pkg/tests/test_krylov.py) run through the
device engine, plus fixed-budget parity with the reference iteration and batch invariance."""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from golden_util import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import FluidProps, assemble_mode_system  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems  # noqa: E402
from paper_2009_06725_b200.krylov import (  # noqa: E402
    SolverSettings, gmres, gmres_batched, gmres_solve, jacobi_precondition,
)
from paper_2009_06725_b200.workloads import C1_TOL, c1_case  # noqa: E402


def _random_complex_symmetric(n, rng):
    m = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    m = 0.5 * (m + m.T)
    m += n * np.eye(n)
    return m


def test_settings_validation():
    with pytest.raises(ValueError):
        SolverSettings(tolerance=2.0)
    with pytest.raises(ValueError):
        SolverSettings(restart=0)
    with pytest.raises(ValueError):
        SolverSettings(preconditioner="ilu")


def test_identity_solved_in_one_iteration():
    a = sp.identity(6, format="csr", dtype=complex)
    b = np.zeros(6, dtype=complex)
    b[0] = 1.0
    x, rep = gmres_solve((a, b), SolverSettings(tolerance=1e-12))
    assert rep.iterations == 1
    assert np.allclose(x, b)


def test_two_by_two_diagonal_complex():
    a = sp.csr_matrix(np.diag([2.0 + 1j, 1.0 - 1j]))
    x, rep = gmres_solve((a, np.array([1.0, 1.0], complex)), SolverSettings(tolerance=1e-13))
    assert x[0] == pytest.approx((2.0 - 1j) / 5.0, rel=1e-12)
    assert x[1] == pytest.approx((1.0 + 1j) / 2.0, rel=1e-12)
    assert rep.converged


def test_manufactured_solution_accuracy():
    rng = np.random.default_rng(3)
    dense = _random_complex_symmetric(40, rng)
    xk = rng.normal(size=40) + 1j * rng.normal(size=40)
    x, rep = gmres_solve((sp.csr_matrix(dense), dense @ xk), SolverSettings(tolerance=1e-12, restart=40))
    assert rep.converged
    assert np.linalg.norm(x - xk) / np.linalg.norm(xk) <= 10.0 * np.linalg.cond(dense) * 1e-12


def test_matches_real_equivalent_system():
    rng = np.random.default_rng(11)
    n = 25
    dense = _random_complex_symmetric(n, rng)
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    big = np.block([[dense.real, -dense.imag], [dense.imag, dense.real]])
    xy = np.linalg.solve(big, np.concatenate([b.real, b.imag]))
    x, rep = gmres_solve((sp.csr_matrix(dense), b), SolverSettings(tolerance=1e-13, restart=60))
    assert rep.converged
    assert np.linalg.norm(x - (xy[:n] + 1j * xy[n:])) / np.linalg.norm(xy) < 1e-10


def test_zero_rhs_early_return():
    x, rep = gmres_solve((sp.identity(4, format="csr", dtype=complex), np.zeros(4, complex)), SolverSettings())
    assert rep.iterations == 0 and rep.converged and np.all(x == 0)


def test_zero_rhs_ignores_x0():
    x, it, hist, conv = gmres(sp.identity(4, format="csr", dtype=complex), np.zeros(4, complex), x0=np.ones(4))
    assert it == 0 and conv and np.all(x == 0) and hist == []


def test_jacobi_rules():
    scale = jacobi_precondition(sp.csr_matrix(np.array([[4.0, 1.0], [1.0, 0.0]], dtype=complex)))
    assert scale[0] == 0.25 and scale[1] == 1.0
    d = np.array([3.0, 5.0 + 2j, 0.5], dtype=complex)
    x, rep = gmres_solve((sp.csr_matrix(np.diag(d)), np.array([1.0, 2.0, 3.0], complex)), SolverSettings(tolerance=1e-13))
    assert rep.iterations == 1
    assert np.allclose(x, np.array([1.0, 2.0, 3.0]) / d)


def test_preconditioner_does_not_slow_convergence():
    rng = np.random.default_rng(5)
    n = 300
    m = rng.normal(size=(n, n))
    dense = np.diag(np.logspace(0, 4, n)) + 0.001 * (m @ m.T)
    b = rng.normal(size=n).astype(complex)
    a = sp.csr_matrix(dense.astype(complex))
    _, plain = gmres_solve((a, b), SolverSettings(tolerance=1e-10, preconditioner="none", restart=50))
    _, jac = gmres_solve((a, b), SolverSettings(tolerance=1e-10, preconditioner="jacobi", restart=50))
    assert plain.converged and jac.converged
    assert jac.iterations <= plain.iterations


def test_history_monotone_within_cycle_and_matches_oracle():
    rng = np.random.default_rng(9)
    dense = _random_complex_symmetric(50, rng)
    b = rng.normal(size=50).astype(complex)
    a = sp.csr_matrix(dense)
    x, iters, hist, conv = gmres(a, b, tol=1e-12, restart=15, maxiter=500)
    assert conv
    for s in range(0, len(hist), 15):
        cyc = hist[s:s + 15]
        assert all(p >= q - 1e-14 for p, q in zip(cyc, cyc[1:]))
    xo, io, ho, co = oracle.gmres(a, b, 1e-12, 15, 500)
    assert iters == io and len(hist) == len(ho)
    np.testing.assert_allclose(hist, ho, rtol=1e-6)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


def test_restarted_path_still_converges():
    rng = np.random.default_rng(13)
    dense = _random_complex_symmetric(80, rng)
    b = rng.normal(size=80).astype(complex)
    x, rep = gmres_solve((sp.csr_matrix(dense), b), SolverSettings(tolerance=1e-10, restart=7))
    assert rep.converged and rep.residual <= 1e-10


def test_initial_guess_used():
    rng = np.random.default_rng(17)
    dense = _random_complex_symmetric(30, rng)
    b = rng.normal(size=30).astype(complex)
    x, rep = gmres_solve((sp.csr_matrix(dense), b), SolverSettings(tolerance=1e-10), x0=np.linalg.solve(dense, b))
    assert rep.iterations <= 1 and rep.converged


def test_maxiter_zero_and_small():
    a = sp.csr_matrix(_random_complex_symmetric(20, np.random.default_rng(2)))
    b = np.ones(20, complex)
    x, it, hist, conv = gmres(a, b, tol=1e-12, maxiter=0)
    assert it == 0 and not conv and np.all(x == 0)
    x, it, hist, conv = gmres(a, b, tol=1e-14, restart=5, maxiter=7)
    xo, io, ho, co = oracle.gmres(a, b, 1e-14, 5, 7)
    assert it == io == 7 and len(hist) == len(ho)
    assert np.linalg.norm(x - xo) <= 1e-10 * np.linalg.norm(xo)


def test_true_residual_contract_on_assembled_system(small_channel_qmesh, fluid):
    system = assemble_mode_system(small_channel_qmesh, fluid, 0.0, h_mode={"inlet": np.array([1.0, 0.0])})
    x, rep = gmres_solve(system, SolverSettings(tolerance=1e-6))
    assert rep.converged
    res = np.linalg.norm(system.rhs - system.matrix @ x) / np.linalg.norm(system.rhs)
    assert res <= 1e-6
    assert rep.residual == pytest.approx(res, rel=1e-10)


def test_deterministic_given_identical_inputs(small_channel_qmesh, fluid):
    system = assemble_mode_system(small_channel_qmesh, fluid, 2.0, h_mode={"inlet": np.array([1.0, 0.0])})
    x1, r1 = gmres_solve(system, SolverSettings(tolerance=1e-8))
    x2, r2 = gmres_solve(system, SolverSettings(tolerance=1e-8))
    assert np.array_equal(x1, x2) and r1.iterations == r2.iterations


def test_homogeneous_problem_has_zero_solution(small_channel_qmesh, fluid):
    system = assemble_mode_system(small_channel_qmesh, fluid, 1.0)
    assert np.linalg.norm(system.rhs) == 0.0
    x, rep = gmres_solve(system, SolverSettings())
    assert rep.converged and np.linalg.norm(x) == 0.0


def test_steady_channel_reproduces_parabola(fluid):
    from paper_2009_06725_b200.mesh import promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid

    q = promote_to_quadratic(channel_grid(8, 4, length=4.0, half_height=1.0))
    system = assemble_mode_system(q, fluid, 0.0, h_mode={"inlet": np.array([1.0, 0.0])})
    x, rep = gmres_solve(system, SolverSettings(tolerance=1e-12))
    assert rep.converged
    u, _ = system.expand(x)
    exact = (1.0 / (2.0 * fluid.viscosity * 4.0)) * (1.0 - q.nodes[:, 1] ** 2)
    assert np.abs(u[:, 0].real - exact).max() / np.abs(exact).max() < 1e-8
    assert np.abs(u[:, 1]).max() < 1e-8


def test_dirichlet_lift_enters_continuity_rows(fluid):
    from paper_2009_06725_b200.mesh import BoundaryPatch, Mesh, promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid

    mesh = channel_grid(4, 3, length=2.0, half_height=1.0)
    patches = dict(mesh.boundary_patches)
    for name in ("inlet", "outlet"):
        patches[name] = BoundaryPatch(kind="dirichlet", faces=patches[name].faces)
    q = promote_to_quadratic(Mesh(mesh.nodes, mesh.elements, patches))
    g = np.zeros((q.n_velocity_nodes, 2), complex)
    prof = 1.0 - q.nodes[:, 1] ** 2
    for name in ("inlet", "outlet"):
        nodes = np.unique(q.boundary_patches[name].face_conn)
        g[nodes, 0] = prof[nodes]
    system = assemble_mode_system(q, fluid, 0.0, g_mode=g)
    assert system.pinned_pressure
    assert np.abs(system.rhs[system.n_velocity_dofs:]).max() > 0.0
    ref = oracle.assemble_mode_system(q, fluid.density, fluid.viscosity, 0.0, g_mode=g)
    assert np.abs(system.rhs - ref.rhs).max() <= 1e-14 * np.abs(ref.rhs).max()
    x, rep = gmres_solve(system, SolverSettings(tolerance=1e-12))
    assert rep.converged
    u, _ = system.expand(x)
    assert np.abs(u[:, 0].real - prof).max() < 1e-7


@pytest.fixture(scope="module")
def c1():
    case = c1_case()
    return case, FluidProps(case.density, case.viscosity), golden("c1.npz")


def test_fixed_budget_cycle_matches_reference(c1):
    """One restart cycle (200 iterations) at c1: estimate history and iterate vs the reference."""
    case, props, g = c1
    s = assemble_mode_system(case.qmesh, props, case.omegas[1], h_mode=case.h_modes()[1])
    x, rep = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=200, max_iterations=200))
    ref_h = g["budget_hist"]
    assert rep.iterations == 200 and len(rep.residual_history) == len(ref_h)
    np.testing.assert_allclose(rep.residual_history, ref_h, rtol=1e-6)
    assert np.linalg.norm(x - g["budget_x"]) <= 1e-8 * np.linalg.norm(g["budget_x"])
    x, rep = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=40, max_iterations=100))
    np.testing.assert_allclose(rep.residual_history, g["budget40_hist"], rtol=1e-6)
    assert np.linalg.norm(x - g["budget40_x"]) <= 1e-8 * np.linalg.norm(g["budget40_x"])


def test_batch_composition_and_order_bitwise(c1):
    """Per-mode results are bitwise independent of which modes share the batch and of their order."""
    case, props, g = c1
    settings = SolverSettings(tolerance=1e-6, restart=30, max_iterations=300)
    idx = [1, 4, 7]
    h = case.h_modes()
    full = assemble_mode_systems(case.qmesh, props, case.omegas[idx], None, [h[i] for i in idx])
    X, rep = gmres_batched(full, settings)
    X = X.cpu().numpy()
    rev = assemble_mode_systems(case.qmesh, props, case.omegas[idx[::-1]], None, [h[i] for i in idx[::-1]])
    Xr, repr_ = gmres_batched(rev, settings)
    Xr = Xr.cpu().numpy()[::-1]
    for j, i in enumerate(idx):
        single = assemble_mode_systems(case.qmesh, props, case.omegas[[i]], None, [h[i]])
        Xs, reps = gmres_batched(single, settings)
        assert np.array_equal(X[j], Xs.cpu().numpy()[0])
        assert np.array_equal(X[j], Xr[j])
        assert rep[j].iterations == reps[0].iterations


@pytest.mark.gpu
def test_maximum_restart_matches_oracle(c1):
    """restart = MAX_RESTART (240): the widest basis-pass instantiations (J up to 241 vectors,
    32 columns per thread, one-stage ring) and the largest triangular solve, checked against the
    oracle's CGS2 GMRES on the same matrix over one full restart cycle plus a few iterations."""
    from oracle import scvs
    from paper_2009_06725_b200.krylov import MAX_RESTART

    case, props, _ = c1
    s = assemble_mode_system(case.qmesh, props, case.omegas[2], h_mode=case.h_modes()[2])
    budget = MAX_RESTART + 10
    x, rep = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=MAX_RESTART, max_iterations=budget))
    a = s.matrix
    xo, it, hist, _ = scvs.gmres(a, s.rhs, C1_TOL, MAX_RESTART, budget, scvs.jacobi_scale(a))
    assert rep.iterations == it == budget
    np.testing.assert_allclose(rep.residual_history, hist, rtol=1e-6)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.gpu
def test_more_modes_than_one_device_batch(c1):
    """gmres_batched chunks beyond MAX_BATCH modes; results equal the per-chunk solves bit for bit."""
    import paper_2009_06725_b200.krylov as K

    case, props, _ = c1
    settings = SolverSettings(tolerance=1e-6, restart=20, max_iterations=60)
    h = case.h_modes()
    idx = [1, 2, 3, 4, 5]
    full = assemble_mode_systems(case.qmesh, props, case.omegas[idx], None, [h[i] for i in idx])
    old = K.MAX_BATCH
    try:
        K.MAX_BATCH = 2   # force chunking into 2 + 2 + 1
        Xc, rc = gmres_batched(full, settings)
    finally:
        K.MAX_BATCH = old
    X, r = gmres_batched(full, settings)
    assert np.array_equal(Xc.cpu().numpy(), X.cpu().numpy())
    assert [a.iterations for a in rc] == [b.iterations for b in r]


@pytest.mark.gpu
@pytest.mark.parametrize("restart", [241, 300])
def test_wide_restart_matches_oracle(c1, restart):
    """restart > 240 (the reference accepts any restart >= 1, krylov.py:24,31-32): the wide basis
    passes (no shared-memory ring, dots in 256-column tiles, Givens/solve staging in global memory)
    against the oracle's CGS2 GMRES over one full cycle plus a few iterations of the next."""
    from oracle import scvs

    case, props, _ = c1
    s = assemble_mode_system(case.qmesh, props, case.omegas[3], h_mode=case.h_modes()[3])
    budget = restart + 7
    x, rep = gmres_solve(s, SolverSettings(tolerance=C1_TOL, restart=restart, max_iterations=budget))
    a = s.matrix
    xo, it, hist, _ = scvs.gmres(a, s.rhs, C1_TOL, restart, budget, scvs.jacobi_scale(a))
    assert rep.iterations == it == budget
    np.testing.assert_allclose(rep.residual_history, hist, rtol=1e-6)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.gpu
def test_wide_restart_converges_generic_csr():
    """gmres(matrix, ...) with restart 600 on a generic complex CSR: converged like the oracle."""
    from oracle import scvs

    rng = np.random.default_rng(21)
    n = 700
    a = sp.random(n, n, density=0.01, random_state=np.random.RandomState(4), dtype=float)
    a = (a + 1j * sp.random(n, n, density=0.01, random_state=np.random.RandomState(5))).tocsr()
    a = a + sp.diags(3.0 + rng.random(n))
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    sc = scvs.jacobi_scale(a)
    x, it, hist, conv = gmres(a, b, tol=1e-11, restart=600, maxiter=2000, scale=sc)
    xo, ito, histo, convo = scvs.gmres(a, b, 1e-11, 600, 2000, sc)
    assert conv and convo and it == ito
    np.testing.assert_allclose(hist, histo, rtol=1e-6)
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


@pytest.mark.gpu
def test_wide_restart_through_solve_modes():
    """solve_modes with SolverSettings(restart=320) converges to the reference's fields (c1 mode 4)."""
    from paper_2009_06725_b200 import solve_mode_systems

    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    g = golden("c1.npz")
    sols = solve_mode_systems(case.qmesh, props, [4], case.omegas[[4]], None, [case.h_modes()[4]],
                              SolverSettings(tolerance=C1_TOL, restart=320))
    s = sols[0]
    assert s.report.converged
    assert np.linalg.norm(s.velocity - g["u_4"]) <= 1e-7 * np.linalg.norm(g["u_4"])


@pytest.mark.gpu
def test_per_mode_wall_time_follows_completion_tick(c1):
    """SolveReport.wall_time per mode: the batch's wall time scaled by the tick at which the mode
    finished (ss_krylov_done_ticks), so a mode needing more iterations reports more time."""
    case, props, _ = c1
    idx = [1, 3, 8]
    h = case.h_modes()
    b = assemble_mode_systems(case.qmesh, props, case.omegas[idx], None, [h[i] for i in idx])
    X, reps = gmres_batched(b, SolverSettings(tolerance=1e-9, restart=50))
    walls = [r.wall_time for r in reps]
    its = [r.iterations for r in reps]
    assert all(w > 0 for w in walls)
    order = np.argsort(its)
    assert all(walls[order[i]] <= walls[order[i + 1]] + 1e-12 for i in range(len(idx) - 1))
    assert max(walls) > 2 * min(walls) or max(its) < 1.5 * min(its)


@pytest.mark.gpu
def test_maximum_batch_with_zero_and_steady_modes(small_channel_qmesh, fluid):
    """MAX_BATCH (256) modes in one call -- steady (omega = 0), zero right-hand sides and ordinary
    modes mixed, solved as concurrent sub-batches -- each equal bit for bit to its own one-mode
    solve (batch invariance at the maximum batch)."""
    from paper_2009_06725_b200.krylov import MAX_BATCH, concurrent_groups

    q = small_channel_qmesh
    nb = MAX_BATCH
    rng = np.random.default_rng(12)
    omegas = np.where(np.arange(nb) % 17 == 0, 0.0, rng.uniform(0.0, 40.0, nb))
    amp = rng.normal(size=nb) + 1j * rng.normal(size=nb)
    amp[5::31] = 0.0                                   # zero traction -> zero rhs -> early return
    h = [{"inlet": a * np.array([1.0, 0.0], complex)} for a in amp]
    settings = SolverSettings(tolerance=1e-8, restart=30, max_iterations=3000)
    batch = assemble_mode_systems(q, fluid, omegas, None, h)
    assert concurrent_groups(batch.operator.n, nb) > 1
    X, reps = gmres_batched(batch, settings)
    X = X.cpu().numpy()
    for b in list(range(0, nb, 23)) + [5, 36]:
        one = assemble_mode_systems(q, fluid, omegas[[b]], None, [h[b]])
        Xs, rs = gmres_batched(one, settings)
        assert np.array_equal(X[b], Xs.cpu().numpy()[0]), b
        assert reps[b].iterations == rs[0].iterations
    for b in range(5, nb, 31):
        assert reps[b].iterations == 0 and reps[b].converged and not np.any(X[b])
    assert all(r.converged for r in reps)


def test_zero_denominator_breakdown_matches_oracle():
    """A x = b with A = 0 (explicit zeros): w = 0, h_kk = h_{k+1,k} = 0, so the Givens denominator is
    0 -- the reference's breakdown branch (krylov.py:124-129): one iteration counted, no update, not
    converged, x = 0 (and the true residual 1)."""
    n = 12
    a = sp.csr_matrix((np.zeros(n, complex), np.arange(n), np.arange(n + 1)), shape=(n, n))
    b = np.arange(1, n + 1) + 0.5j
    x, it, hist, conv = gmres(a, b, tol=1e-10, restart=5, maxiter=50)
    xo, io, ho, co = oracle.gmres(a, b, 1e-10, 5, 50)
    assert it == io == 1 and not conv and not co
    assert hist == ho == []
    assert np.all(x == 0) and np.all(xo == 0)


@pytest.mark.parametrize("n", [1, 37])
def test_restart_one_and_tiny_systems_match_oracle(n):
    """GMRES(1) (every iteration a cycle end) and a 1x1 system, against the oracle iteration."""
    rng = np.random.default_rng(40 + n)
    a = sp.csr_matrix(_random_complex_symmetric(n, rng))
    b = rng.normal(size=n) + 1j * rng.normal(size=n)
    sc = oracle.jacobi_scale(a)
    x, it, hist, conv = gmres(a, b, tol=1e-11, restart=1, maxiter=400, scale=sc)
    xo, io, ho, co = oracle.gmres(a, b, 1e-11, 1, 400, scale=sc)
    assert it == io and conv == co
    # estimates agree to rounding relative to the initial (preconditioned) residual norm: the last
    # ones sit at 1e-13 of it (n = 37), or at the 1e-32 noise floor of an exact 1-step solve (n = 1)
    np.testing.assert_allclose(hist, ho, rtol=1e-6, atol=1e-10 * np.linalg.norm(sc * b))
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
