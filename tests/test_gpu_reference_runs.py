"""GPU runs pinned to fixtures the REFERENCE produced (tests/golden/make_golden.py):

* config 2 at full size (199 800 jittered tets, n = 796 978): one fixed-budget restart cycle of
  GMRES(200) from x0 = 0 for modes 1 and 16 (reference krylov.py:63-164, ~125 s of CPU per mode):
  the per-iteration residual estimates, the iterate at 20 000 sampled rows, ||x|| and four
  projections of x onto seeded complex vectors (c2_gmres.npz);
* adaptive_mode_refinement (reference spectral.py:333-371) on seeded sampled waveforms: the final
  N_m, the converged flag and the number of solved modes exactly, per-mode energies and the last
  solved velocity field to tolerance (adaptive.npz).
"""

import numpy as np
import pytest

from golden_util import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import (  # noqa: E402
    BoundaryWaveform, FluidProps, SolverSettings, adaptive_mode_refinement, mode_energies,
)
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.krylov import gmres_batched  # noqa: E402
from paper_2009_06725_b200.mesh import promote_to_quadratic  # noqa: E402
from paper_2009_06725_b200.structured import channel_grid  # noqa: E402
from paper_2009_06725_b200.workloads import c2_case  # noqa: E402

MODES = (1, 16)


def test_config2_fixed_budget_cycle_matches_reference():
    g = golden("c2_gmres.npz")
    case = c2_case()
    q = case.qmesh
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(q, props)
    assert op.n == int(g["n_1"])
    batch = assemble_mode_systems(q, props, case.omegas[list(MODES)],
                                  [case.coefficients[i] * case.profile for i in MODES], None, operator=op)
    X, reps = gmres_batched(batch, SolverSettings(tolerance=1e-10, restart=200, max_iterations=200))
    X = X.cpu().numpy()
    for j, m in enumerate(MODES):
        x = X[j, : op.n]
        rep = reps[j]
        assert rep.iterations == int(g[f"iters_{m}"]) == 200
        assert not rep.converged and not bool(g[f"conv_{m}"])
        np.testing.assert_allclose(rep.residual_history, g[f"hist_{m}"], rtol=1e-6)
        xr = g[f"x_rows_{m}"]
        assert np.linalg.norm(x[g[f"rows_{m}"]] - xr) <= 1e-8 * np.linalg.norm(xr)
        assert np.linalg.norm(x) == pytest.approx(float(g[f"x_norm_{m}"]), rel=1e-9)
        rng = np.random.default_rng(2000 + m)
        proj = np.stack([rng.normal(size=op.n) + 1j * rng.normal(size=op.n) for _ in range(4)]) @ x
        assert np.abs(proj - g[f"proj_{m}"]).max() <= 1e-8 * np.abs(g[f"proj_{m}"]).max()
        assert rep.residual == pytest.approx(float(g[f"res_{m}"]), rel=1e-8)


# same cases as tests/golden/make_golden.py ADAPTIVE_CASES / adaptive_signal
CASES = {
    "square": ("square", 10.0, 1e-3, 12),
    "saw": ("saw", 1.0, 1e-2, 20),
    "saw_cap": ("saw", 1.0, 2e-3, 16),
    "noisy": ("noisy", 10.0, 1e-2, 16),
}


def _signal(kind, n=128):
    t = np.arange(n) / n
    if kind == "square":
        return np.where(t < 0.5, 1.0, -1.0)
    if kind == "saw":
        return t - 0.5
    rng = np.random.default_rng(333)
    return np.sin(2 * np.pi * t) + 0.3 * np.sin(6 * np.pi * t + 0.4) + 0.2 * rng.normal(size=n)


@pytest.mark.parametrize("name", sorted(CASES))
def test_adaptive_refinement_matches_reference(name):
    g = golden("adaptive.npz")
    sig, period, tol, mm = CASES[name]
    q = promote_to_quadratic(channel_grid(6, 3, length=2.0, half_height=1.0))
    props = FluidProps(1.0, 1.0)
    wf = BoundaryWaveform(patch="inlet", kind="neumann", direction=np.array([1.0, 0.0]), period=period,
                          samples=_signal(sig))
    sols, final_nm, conv = adaptive_mode_refinement(q, props, [wf], tol, SolverSettings(tolerance=1e-10),
                                                    max_modes=mm)
    assert final_nm == int(g[f"{name}_final_nm"])
    assert conv == bool(g[f"{name}_converged"])
    assert len(sols) == int(g[f"{name}_n_solved"])
    e = mode_energies(sols, q, period)
    ref = g[f"{name}_energies"]
    scale = ref.max()
    assert np.abs(e - ref).max() <= 1e-9 * scale
    u = sols[-1].velocity
    ur = g[f"{name}_u_last"]
    assert np.linalg.norm(u - ur) <= 1e-7 * max(np.linalg.norm(ur), 1e-300) or np.linalg.norm(ur) == 0.0


def test_config3_full_size_fixed_budget_matches_reference():
    """Config 3 at full size (2 059 200-tet bend, n = 8.39 M): 40 iterations of GMRES(40) from x0 = 0
    for mode 1 against the reference's own run (tests/golden/c3_gmres.npz): pattern SHA, history,
    sampled iterate, ||x|| and projections."""
    import hashlib

    from paper_2009_06725_b200.workloads import c3_case

    g = golden("c3_gmres.npz")
    case = c3_case()
    q = case.qmesh
    props = FluidProps(case.density, case.viscosity)
    op = get_operator(q, props)
    assert op.n == int(g["n"]) and op.nnz == int(g["nnz"])
    ip, ix = op.pattern()
    h = hashlib.sha256()
    for a in (ip, ix):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(g["pattern_sha"])
    batch = assemble_mode_systems(q, props, case.omegas[[1]], [case.coefficients[1] * case.profile], None, operator=op)
    X, reps = gmres_batched(batch, SolverSettings(tolerance=1e-10, restart=40, max_iterations=40))
    x = X[0, : op.n].cpu().numpy()
    assert reps[0].iterations == int(g["iters"]) == 40
    np.testing.assert_allclose(reps[0].residual_history, g["hist"], rtol=1e-6)
    assert np.linalg.norm(x[g["rows"]] - g["x_rows"]) <= 1e-8 * np.linalg.norm(g["x_rows"])
    assert np.linalg.norm(x) == pytest.approx(float(g["x_norm"]), rel=1e-9)
    rng = np.random.default_rng(2301)
    proj = np.stack([rng.normal(size=op.n) + 1j * rng.normal(size=op.n) for _ in range(2)]) @ x
    assert np.abs(proj - g["proj"]).max() <= 1e-8 * np.abs(g["proj"]).max()
    op.release_workspaces()
