"""Structural properties of the assembled complex saddle system and the solved fields, as the
reference checks them in pkg/tests/test_assembly.py:113-275 and test_spectral.py:137-145,
restated against the device-assembled operator."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import (  # noqa: E402
    BoundaryWaveform, SolverSettings, assemble_mode_system, fourier_transform_bcs, gmres_solve,
    promote_to_quadratic, solve_modes,
)
from paper_2009_06725_b200.structured import channel_grid  # noqa: E402

TRACTION = {"inlet": np.array([1.0, 0.0])}


def test_matrix_is_complex_symmetric(small_channel_qmesh, fluid):
    a = assemble_mode_system(small_channel_qmesh, fluid, 2.0 * np.pi, h_mode=TRACTION).matrix
    d = (a - a.T).tocoo()
    assert (np.max(np.abs(d.data)) if d.nnz else 0.0) <= 1e-13 * np.max(np.abs(a.data))


def test_pressure_block_is_empty(small_channel_qmesh, fluid):
    s = assemble_mode_system(small_channel_qmesh, fluid, 2.0, h_mode=TRACTION)
    nu = s.n_velocity_dofs
    blk = s.matrix.tocsc()[nu:, nu:]
    assert blk.nnz == 0 or np.max(np.abs(blk.data)) == 0.0


def test_dirichlet_data_off_constrained_nodes_is_rejected(small_channel_qmesh, fluid):
    q = small_channel_qmesh
    interior = np.setdiff1d(np.arange(q.n_velocity_nodes), np.unique(q.boundary_patches["walls"].face_conn))
    g = np.zeros((q.n_velocity_nodes, 2), dtype=complex)
    g[interior[0]] = 1.0
    with pytest.raises(ValueError, match="Dirichlet"):
        assemble_mode_system(q, fluid, 0.0, g_mode=g)


def test_velocity_block_rayleigh_quotients(small_channel_qmesh, fluid):
    s = assemble_mode_system(small_channel_qmesh, fluid, 3.0, h_mode=TRACTION)
    nu = s.n_velocity_dofs
    a = s.matrix.tocsc()[:nu, :nu]
    rng = np.random.default_rng(5)
    for _ in range(5):
        v = rng.normal(size=nu) + 1j * rng.normal(size=nu)
        rq = np.vdot(v, a @ v)
        assert rq.real > 0.0 and rq.imag > 0.0     # viscous (SPD) + omega * mass (SPD)


def test_wall_reactions_balance_the_applied_traction(fluid):
    q = promote_to_quadratic(channel_grid(8, 4, length=4.0, half_height=1.0))
    s = assemble_mode_system(q, fluid, 0.0, h_mode=TRACTION)
    x, rep = gmres_solve(s, SolverSettings(tolerance=1e-12))
    assert rep.converged
    net = s.reaction_forces(x).reshape(-1, 2).sum(axis=0)
    assert net[0].real == pytest.approx(-2.0, rel=1e-9)   # traction 1 over the inlet of length 2
    assert abs(net[1]) < 1e-9


def test_matrix_export_round_trips(tmp_path, small_channel_qmesh, fluid):
    s = assemble_mode_system(small_channel_qmesh, fluid, 1.0, h_mode=TRACTION)
    path = tmp_path / "a.txt"
    s.export_matrix(path)
    lines = path.read_text().splitlines()[1:]
    coo = s.matrix.tocoo()
    assert len(lines) == coo.nnz
    for k in (0, 137 % len(lines), len(lines) - 1):
        r, c, re, im = lines[k].split()
        assert s.matrix[int(r), int(c)] == complex(float(re), float(im))


def test_steady_only_mode_set(small_channel_qmesh, fluid):
    w = BoundaryWaveform(patch="inlet", kind="neumann", direction=np.array([1.0, 0.0]), period=1.0,
                         coefficients=np.array([1.0], dtype=complex))
    sols = solve_modes(small_channel_qmesh, fluid, fourier_transform_bcs([w], 0), SolverSettings(tolerance=1e-9))
    assert len(sols) == 1 and sols[0].omega == 0.0 and sols[0].report.converged
    assert np.max(np.abs(sols[0].velocity.imag)) < 1e-12
