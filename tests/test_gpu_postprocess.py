"""GPU post-processing: L2 norms / mode energies and adaptive refinement,
against the oracle restatement of metrics.py:12-18 and the reference's adaptive tests
(pkg/tests/test_spectral.py:222-257)."""

import numpy as np
import pytest

import oracle
from golden_util import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import (  # noqa: E402
    BoundaryWaveform, SolverSettings, adaptive_mode_refinement, l2_norm, l2_norms, mode_energies,
)
from paper_2009_06725_b200.krylov import SolveReport  # noqa: E402
from paper_2009_06725_b200.spectral import ModeSolution  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, pipe3d_case  # noqa: E402

SETTINGS = SolverSettings(tolerance=1e-9)


def _wave(values=None, coeffs=None, period=1.0):
    return BoundaryWaveform(patch="inlet", kind="neumann", direction=np.array([1.0, 0.0]), period=period,
                            samples=None if values is None else np.asarray(values, float),
                            coefficients=None if coeffs is None else np.asarray(coeffs, complex))


def test_l2_norm_matches_oracle_2d_and_3d():
    g = golden("c1.npz")
    q = c1_case().qmesh
    fields = np.stack([g[f"u_{i}"] for i in range(9)])
    dev = l2_norms(fields, q)
    for i in range(9):
        assert dev[i] == pytest.approx(oracle.l2_norm(fields[i], q), rel=1e-12)
    assert l2_norm(fields[3][:, 0].real, q) == pytest.approx(oracle.l2_norm(fields[3][:, 0].real, q), rel=1e-12)
    p3 = golden("pipe3d.npz")
    q3 = pipe3d_case().qmesh
    assert l2_norm(p3["u_16"], q3) == pytest.approx(oracle.l2_norm(p3["u_16"], q3), rel=1e-12)


def test_mode_energies_time_weights():
    g = golden("c1.npz")
    q = c1_case().qmesh
    sols = [ModeSolution(i, float(g["omegas"][i]), g[f"u_{i}"], g[f"p_{i}"], SolveReport(0, 0.0, True, 0.0))
            for i in range(3)]
    e = mode_energies(sols, q, 2.0)
    for i, s in enumerate(sols):
        w = 2.0 if i == 0 else 1.0
        assert e[i] == pytest.approx(w * oracle.l2_norm(s.velocity, q) ** 2, rel=1e-12)


def test_adaptive_stops_at_band_limit(small_channel_qmesh, fluid):
    sols, final_nm, converged = adaptive_mode_refinement(small_channel_qmesh, fluid, [_wave(coeffs=[0.4, 1.0, 0.5])],
                                                         1e-10, SETTINGS)
    assert converged and final_nm == 2


def test_adaptive_loose_tolerance_stops_immediately(small_channel_qmesh, fluid):
    sols, final_nm, converged = adaptive_mode_refinement(small_channel_qmesh, fluid, [_wave(coeffs=[1.0, 0.5, 0.25])],
                                                         0.9, SETTINGS)
    assert converged and final_nm == 1 and len(sols) == 2


def test_adaptive_square_wave_differences_decrease(fluid):
    from paper_2009_06725_b200.mesh import promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid

    q = promote_to_quadratic(channel_grid(6, 3, length=2.0, half_height=1.0))
    t = np.arange(128) / 128
    wf = _wave(values=np.where(t < 0.5, 1.0, -1.0), period=10.0)
    sols, final_nm, _ = adaptive_mode_refinement(q, fluid, [wf], 1e-4, SETTINGS, max_modes=9)
    diffs = [np.sqrt(0.5 * wf.period) * l2_norm(s.velocity, q) for s in sols[1:] if s.omega != 0]
    nonzero = [d for d in diffs if d > 0]
    assert all(a > b for a, b in zip(nonzero, nonzero[1:]))
    # the adaptive result equals solving the same modes directly
    ref = [np.sqrt(0.5 * wf.period) * oracle.l2_norm(s.velocity, q) for s in sols[1:] if s.omega != 0]
    np.testing.assert_allclose(diffs, ref, rtol=1e-12)


def _post_oracle(xy):
    """Same analytic point field as tests/golden/make_golden.py:post_oracle."""
    x = np.asarray(xy, dtype=float)
    cols = [np.sin(1.3 * x[:, 0]) + 0.5j * x[:, 1] ** 2, np.cos(0.7 * x[:, 1]) - 0.25j * x[:, 0]]
    if x.shape[1] == 3:
        cols.append(x[:, 2] * x[:, 0] + 1j * np.sin(x[:, 2]))
    return np.stack(cols, axis=1)


@pytest.mark.parametrize("name", ["c1", "pipe3d"])
def test_interpolate_at_quadrature_and_field_error_match_reference(name):
    """Device interpolation (assembly.py:497-511) and field_error / l2_norm (metrics.py:12-39)
    against the reference's own outputs on the same meshes and seeded fields."""
    from paper_2009_06725_b200 import field_error, interpolate_at_quadrature

    g = golden("post.npz")
    q = c1_case().qmesh if name == "c1" else pipe3d_case().qmesh
    vec, sca = g[f"{name}_vec"], g[f"{name}_sca"]
    coords, vals, w = interpolate_at_quadrature(q, vec)
    assert coords.shape == g[f"{name}_iq_coords"].shape and vals.shape == g[f"{name}_iq_vals"].shape
    np.testing.assert_allclose(coords, g[f"{name}_iq_coords"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(w, g[f"{name}_iq_w"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(vals, g[f"{name}_iq_vals"], rtol=0, atol=1e-13 * np.abs(vec).max())
    _, svals, _ = interpolate_at_quadrature(q, sca)
    assert not np.iscomplexobj(svals) and svals.shape == g[f"{name}_iq_svals"].shape
    np.testing.assert_allclose(svals, g[f"{name}_iq_svals"], rtol=0, atol=1e-13 * np.abs(sca).max())
    assert l2_norm(vec, q) == pytest.approx(float(g[f"{name}_l2_vec"]), rel=1e-12)
    assert field_error(g[f"{name}_near"], _post_oracle, q) == pytest.approx(float(g[f"{name}_field_error"]), rel=1e-9)
    with pytest.raises(ZeroDivisionError):
        field_error(vec, lambda xy: np.zeros((len(xy), q.dim)), q)
