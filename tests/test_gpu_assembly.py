"""GPU parity: pattern, element values, right-hand sides, Jacobi and SpMV against the reference.

All compute goes through the C ABI (libss_b200.so).  Bars: integer patterns bit-exact; values
within 1e-13 * max|A|; SpMV within 1e-13 relative.
"""

import hashlib

import numpy as np
import pytest

import oracle
from golden_util import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2009_06725_b200 import FluidProps, assemble_mode_system, jacobi_precondition  # noqa: E402
from paper_2009_06725_b200.assembly import assemble_mode_systems, get_operator  # noqa: E402
from paper_2009_06725_b200.errors import MeshError  # noqa: E402
from paper_2009_06725_b200.workloads import c1_case, c2_case, pipe3d_case  # noqa: E402


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def c1():
    case = c1_case()
    props = FluidProps(case.density, case.viscosity)
    return case, props, golden("c1.npz")


def test_c1_pattern_bit_exact(c1):
    case, props, g = c1
    op = get_operator(case.qmesh, props)
    ip, ix = op.pattern()
    assert np.array_equal(ip, g["indptr"]) and np.array_equal(ix, g["indices"])
    vd, pd = op.dof_maps()
    assert np.array_equal(vd, g["vel_dof"]) and np.array_equal(pd, g["pres_dof"])


def test_c1_values_and_rhs(c1):
    case, props, g = c1
    h = case.h_modes()
    s = assemble_mode_system(case.qmesh, props, case.omegas[1], h_mode=h[1])
    ref = g["data_1"]
    scale = np.abs(ref).max()
    assert np.abs(s.matrix.data - ref).max() <= 1e-13 * scale
    np.testing.assert_array_equal(s.matrix.indices, g["indices"])
    for i in range(case.n_modes + 1):
        si = assemble_mode_system(case.qmesh, props, case.omegas[i], h_mode=h[i])
        r = g[f"rhs_{i}"]
        assert np.abs(si.rhs - r).max() <= 1e-14 * max(np.abs(r).max(), 1e-300)
    jac = jacobi_precondition(s)
    np.testing.assert_allclose(jac, g["jacobi_1"], rtol=1e-13)


def test_c1_spmv(c1):
    case, props, g = c1
    op = get_operator(case.qmesh, props)
    x = np.zeros((1, op.ld), complex)
    x[0, : op.n] = g["spmv_x"]
    y = op.spmv([case.omegas[1]], torch.from_numpy(x).cuda()).cpu().numpy()[0, : op.n]
    ref = g["spmv_y"]
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)


def test_spmv_batched_matches_per_mode_oracle(c1):
    case, props, g = c1
    op = get_operator(case.qmesh, props)
    rng = np.random.default_rng(3)
    nb = case.n_modes + 1
    x = np.zeros((nb, op.ld), complex)
    x[:, : op.n] = rng.normal(size=(nb, op.n)) + 1j * rng.normal(size=(nb, op.n))
    y = op.spmv(case.omegas, torch.from_numpy(x).cuda(), jacobi=True).cpu().numpy()
    h = case.h_modes()
    for b in range(nb):
        s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[b], h_mode=h[b])
        ref = oracle.jacobi_scale(s.matrix) * (s.matrix @ x[b, : op.n])
        assert np.linalg.norm(y[b, : op.n] - ref) <= 1e-13 * np.linalg.norm(ref)
        assert np.all(y[b, op.n:] == 0)


def test_pattern_identical_for_all_omega(c1):
    case, props, g = c1
    for om in (0.0, 2 * np.pi, 16 * np.pi):
        s = assemble_mode_system(case.qmesh, props, om, h_mode=case.h_modes()[1])
        assert np.array_equal(s.matrix.indptr, g["indptr"]) and np.array_equal(s.matrix.indices, g["indices"])
        if om == 0.0:
            assert np.abs(s.matrix.data.imag).max() == 0.0


def test_pipe3d_pattern_and_rhs():
    case = pipe3d_case()
    g = golden("pipe3d.npz")
    props = FluidProps(case.density, case.viscosity)
    for idx in (1, 16):
        s = assemble_mode_system(case.qmesh, props, case.omegas[idx], g_mode=case.coefficients[idx] * case.profile)
        assert _sha(s.matrix.indptr, s.matrix.indices) == str(g[f"pattern_sha_{idx}"])
        r = g[f"rhs_{idx}"]
        assert np.abs(s.rhs - r).max() <= 1e-13 * np.abs(r).max()
        ref = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[idx],
                                          g_mode=case.coefficients[idx] * case.profile).matrix
        assert np.abs(s.matrix.data - ref.data).max() <= 1e-13 * np.abs(ref.data).max()


def test_c2_pattern_spmv_rhs_full_size():
    """BASELINE config 2 at full size (199 800 tets): pattern hash, sampled A@x, rhs, diagonal."""
    case = c2_case()
    g = golden("c2_pattern.npz")
    props = FluidProps(case.density, case.viscosity)
    for idx in (0, 1):
        s = assemble_mode_system(case.qmesh, props, case.omegas[idx], g_mode=case.coefficients[idx] * case.profile)
        ip, ix = s.operator.pattern()
        assert _sha(ip, ix) == str(g[f"pattern_sha_{idx}"]) and ix.size == int(g[f"nnz_{idx}"])
        rows = g[f"spmv_rows_{idx}"]
        np.testing.assert_allclose(s.rhs[rows], g[f"rhs_rows_{idx}"], rtol=1e-12, atol=1e-13 * np.abs(g[f"rhs_rows_{idx}"]).max())
        rng = np.random.default_rng(99)
        op = s.operator
        xs = rng.normal(size=op.n) + 1j * rng.normal(size=op.n)
        x = np.zeros((1, op.ld), complex)
        x[0, : op.n] = xs
        y = op.spmv([case.omegas[idx]], torch.from_numpy(x).cuda()).cpu().numpy()[0]
        ref = g[f"spmv_y_{idx}"]
        assert np.abs(y[rows] - ref).max() <= 1e-12 * np.abs(ref).max()
        yn = np.linalg.norm(y[: op.n])
        assert abs(yn - float(g[f"spmv_norm_{idx}"])) <= 1e-12 * yn


def test_batched_rhs_equals_single(c1):
    case, props, g = c1
    h = case.h_modes()
    batch = assemble_mode_systems(case.qmesh, props, case.omegas, None, h)
    rhs = batch.rhs.cpu().numpy()
    for i in range(case.n_modes + 1):
        single = assemble_mode_system(case.qmesh, props, case.omegas[i], h_mode=h[i]).rhs
        assert np.array_equal(rhs[i, : single.size], single)


def test_dirichlet_misuse_and_errors(small_channel_qmesh, fluid):
    q = small_channel_qmesh
    g = np.zeros((q.n_velocity_nodes, 2), complex)
    interior = np.setdiff1d(np.arange(q.n_velocity_nodes), np.unique(q.boundary_patches["walls"].face_conn))
    g[interior[0]] = 1.0
    with pytest.raises(ValueError, match="Dirichlet"):
        assemble_mode_system(q, fluid, 0.0, g_mode=g)
    with pytest.raises(ValueError):
        assemble_mode_system(q, fluid, -1.0)
    with pytest.raises(ValueError):
        assemble_mode_system(q, fluid, 1.0, g_mode=np.zeros((3, 2)))


def test_degenerate_element_raises_mesh_error():
    from paper_2009_06725_b200.mesh import QuadraticMesh, promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid

    q = promote_to_quadratic(channel_grid(2, 2, 1.0, 1.0))
    nodes = q.nodes.copy()
    nodes[q.elements[0, 1]] = nodes[q.elements[0, 0]]   # collapse an element
    bad = QuadraticMesh(nodes, q.n_vertices, q.elements, q.vel_conn, q.edges, q.boundary_patches)
    with pytest.raises(MeshError):
        get_operator(bad, FluidProps(1.0, 1.0))


def test_omega_zero_real_and_symmetric(small_channel_qmesh, fluid):
    s = assemble_mode_system(small_channel_qmesh, fluid, 0.0, h_mode={"inlet": np.array([1.0, 0.0])})
    assert np.abs(s.matrix.toarray().imag).max() == 0.0
    s2 = assemble_mode_system(small_channel_qmesh, fluid, 2 * np.pi, h_mode={"inlet": np.array([1.0, 0.0])})
    d = (s2.matrix - s2.matrix.T).tocoo()
    assert (np.abs(d.data).max() if d.nnz else 0.0) <= 1e-13 * np.abs(s2.matrix.data).max()
    n_u = s2.n_velocity_dofs
    blk = s2.matrix.tocsc()[n_u:, n_u:]
    assert blk.nnz == 0 or np.abs(blk.data).max() == 0.0


def _rows_close(a, b, tol=1e-13):
    a, b = a.tocsr(), b.tocsr()
    assert a.shape == b.shape
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.abs(a.data - b.data).max() <= tol * np.abs(b.data).max()


def test_constrained_rows_and_reaction_forces(fluid):
    """a_full[fixed_idx], rhs_full[fixed_idx] and the momentum balance (assembly.py:364-367,491-492)."""
    from paper_2009_06725_b200.krylov import SolverSettings, gmres_solve
    from paper_2009_06725_b200.mesh import promote_to_quadratic
    from paper_2009_06725_b200.structured import channel_grid

    q = promote_to_quadratic(channel_grid(8, 4, length=4.0, half_height=1.0))
    h = {"inlet": np.array([1.0, 0.0])}
    system = assemble_mode_system(q, fluid, 0.0, h_mode=h)
    ref = oracle.assemble_mode_system(q, fluid.density, fluid.viscosity, 0.0, h_mode=h)
    _rows_close(system.constrained_rows, ref.constrained_rows)
    np.testing.assert_allclose(system.constrained_rhs, ref.constrained_rhs, rtol=1e-14, atol=1e-15)
    x, _ = gmres_solve(system, SolverSettings(tolerance=1e-12))
    total = system.reaction_forces(x).reshape(-1, 2).sum(axis=0)
    assert total[0].real == pytest.approx(-2.0, rel=1e-9)      # reference test_assembly.py:226-236
    assert abs(total[1]) < 1e-9
    s2 = assemble_mode_system(q, fluid, 3.0, h_mode=h)
    _rows_close(s2.constrained_rows, oracle.assemble_mode_system(q, 1.0, 1.0, 3.0, h_mode=h).constrained_rows)


def test_constrained_rows_with_pinned_pressure_3d():
    case = pipe3d_case()
    props = FluidProps(case.density, case.viscosity)
    from paper_2009_06725_b200.mesh import with_patch_kinds, promote_to_quadratic

    m = with_patch_kinds(case.mesh, {"outlet": "dirichlet"})          # no Neumann patch -> pinned
    q = promote_to_quadratic(m, case.geometry)
    g = case.coefficients[2] * case.profile
    s = assemble_mode_system(q, props, case.omegas[2], g_mode=g)
    assert s.pinned_pressure
    ref = oracle.assemble_mode_system(q, case.density, case.viscosity, case.omegas[2], g_mode=g)
    _rows_close(s.constrained_rows, ref.constrained_rows)
    assert np.array_equal(s.matrix.indices, ref.matrix.indices)


def test_interleaved_spmv_matches_row_layout_and_oracle(c1):
    case, props, g = c1
    op = get_operator(case.qmesh, props)
    nb = case.n_modes + 1
    rng = np.random.default_rng(8)
    x = np.zeros((nb, op.ld), complex)
    x[:, : op.n] = rng.normal(size=(nb, op.n)) + 1j * rng.normal(size=(nb, op.n))
    xr = torch.from_numpy(x).cuda()
    y_row = op.spmv(case.omegas, xr, jacobi=True).cpu().numpy()
    y_int = op.spmv_interleaved(case.omegas, xr.t().contiguous(), jacobi=True).cpu().numpy()
    h = case.h_modes()
    for b in range(nb):
        s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[b], h_mode=h[b])
        ref = oracle.jacobi_scale(s.matrix) * (s.matrix @ x[b, : op.n])
        assert np.linalg.norm(y_int[b, : op.n] - ref) <= 1e-13 * np.linalg.norm(ref)
        assert np.linalg.norm(y_int[b, : op.n] - y_row[b, : op.n]) <= 1e-14 * np.linalg.norm(ref)
