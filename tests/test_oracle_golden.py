"""Pin the oracle (CPU restatement) against vectors produced by the reference itself.

Fixtures come from tests/golden/make_golden.py, which imported the reference read-only in the
build container.  These tests need no GPU and never read /root/reference.
"""

import hashlib

import numpy as np
import pytest

import oracle
from paper_2009_06725_b200.workloads import c1_case, c2_case, pipe3d_case
from golden_util import golden


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("dim", [2, 3])
def test_reference_tables_match_reference(dim):
    g = golden("shapes.npz")
    t = oracle.reference_tables(dim)
    for key in ("points", "weights", "vel_values", "vel_grads", "pres_values"):
        assert np.array_equal(getattr(t, key), g[f"d{dim}_{key}"]), key
    np.testing.assert_allclose(t.mref, g[f"d{dim}_mref"], rtol=0, atol=1e-16)
    np.testing.assert_allclose(t.sref, g[f"d{dim}_sref"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(t.tref, g[f"d{dim}_tref"], rtol=0, atol=1e-16)


@pytest.fixture(scope="module")
def c1():
    case = c1_case()
    return case, golden("c1.npz")


def test_c1_mesh_is_the_reference_mesh(c1):
    case, g = c1
    q = case.qmesh
    assert np.array_equal(q.nodes, g["mesh_nodes"])
    assert np.array_equal(q.vel_conn, g["mesh_vel_conn"])
    assert np.array_equal(q.edges, g["mesh_edges"])


def test_c1_assembly_bitwise(c1):
    case, g = c1
    h = case.h_modes()
    s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[1], h_mode=h[1])
    assert np.array_equal(s.matrix.indptr, g["indptr"])
    assert np.array_equal(s.matrix.indices, g["indices"])
    assert np.array_equal(s.matrix.data, g["data_1"])
    assert np.array_equal(s.vel_dof, g["vel_dof"]) and np.array_equal(s.pres_dof, g["pres_dof"])
    assert np.array_equal(oracle.jacobi_scale(s.matrix), g["jacobi_1"])
    for i in range(case.n_modes + 1):
        si = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[i], h_mode=h[i])
        assert np.array_equal(si.rhs, g[f"rhs_{i}"]), i
    assert bool(g["pattern_same_all_omega"])


def test_c1_fixed_budget_gmres(c1):
    """200 iterations (one restart cycle) and 100 iterations at restart 40 reproduce the reference."""
    case, g = c1
    s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[1], h_mode=case.h_modes()[1])
    sc = oracle.jacobi_scale(s.matrix)
    for tag, restart, maxiter in (("budget", 200, 200), ("budget40", 40, 100)):
        x, it, hist, conv = oracle.gmres(s.matrix, s.rhs, 1e-10, restart, maxiter, sc)
        ref_h = g[f"{tag}_hist"]
        assert it == maxiter and len(hist) == len(ref_h)
        np.testing.assert_allclose(hist, ref_h, rtol=1e-9)
        assert np.linalg.norm(x - g[f"{tag}_x"]) <= 1e-12 * np.linalg.norm(g[f"{tag}_x"])


def test_c1_reference_solutions_converged(c1):
    _, g = c1
    for i in range(9):
        assert bool(g[f"conv_{i}"]) and float(g[f"res_{i}"]) <= 1e-10


@pytest.mark.parametrize("j", [0, 1, 2, 3])
def test_c1_reconstruct_matches_reference(c1, j):
    case, g = c1
    vel = [g[f"u_{i}"] for i in range(9)]
    pre = [g[f"p_{i}"] for i in range(9)]
    u, p = oracle.reconstruct(vel, pre, list(g["omegas"]), float(g["recon_t"][j]))
    assert np.array_equal(u, g[f"recon_u_{j}"])
    assert np.array_equal(p, g[f"recon_p_{j}"])


def test_pipe3d_rhs_and_pattern():
    case = pipe3d_case()
    g = golden("pipe3d.npz")
    assert np.array_equal(case.qmesh.nodes, g["mesh_nodes"])
    assert np.array_equal(case.profile, g["profile"])
    for idx in (1, 16):
        s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[idx],
                                        g_mode=case.coefficients[idx] * case.profile)
        assert _sha(s.matrix.indptr, s.matrix.indices) == str(g[f"pattern_sha_{idx}"])
        assert np.array_equal(s.rhs, g[f"rhs_{idx}"])


def test_pipe3d_oracle_solution_short_budget():
    """Oracle GMRES on the 3D system: 60 iterations, residual history strictly decreasing."""
    case = pipe3d_case()
    s = oracle.assemble_mode_system(case.qmesh, case.density, case.viscosity, case.omegas[1],
                                    g_mode=case.coefficients[1] * case.profile)
    x, it, hist, conv = oracle.gmres(s.matrix, s.rhs, 1e-10, 200, 60, oracle.jacobi_scale(s.matrix))
    assert it == 60 and all(a >= b for a, b in zip(hist, hist[1:]))


@pytest.mark.slow
def test_c2_pattern_and_spmv_match_reference():
    """BASELINE config 2 (199 800 jittered tets): pattern hash, sampled A@x and rhs."""
    case = c2_case()
    g = golden("c2_pattern.npz")
    q = case.qmesh
    assert _sha(q.nodes) == str(g["mesh_nodes_sha"]) and _sha(q.vel_conn) == str(g["mesh_conn_sha"])
    rng = np.random.default_rng(99)
    s = oracle.assemble_mode_system(q, case.density, case.viscosity, case.omegas[1],
                                    g_mode=case.coefficients[1] * case.profile)
    assert _sha(s.matrix.indptr, s.matrix.indices) == str(g["pattern_sha_1"])
    x = rng.normal(size=s.matrix.shape[0]) + 1j * rng.normal(size=s.matrix.shape[0])
    rows = g["spmv_rows_1"]
    y = s.matrix @ x
    np.testing.assert_allclose(y[rows], g["spmv_y_1"], rtol=1e-12, atol=1e-12 * np.abs(g["spmv_y_1"]).max())
    np.testing.assert_allclose(s.rhs[rows], g["rhs_rows_1"], rtol=1e-12, atol=1e-14)
