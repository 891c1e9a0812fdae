"""Generate the golden fixtures from the REFERENCE implementation itself.

Run once in the build container (the only place `/root/reference` exists):

    python tests/golden/make_golden.py            # all fixtures (~5 min on 8 cores)

It imports the reference package read-only (`/root/reference/pkg/src/spectralstokes`), never its
CLI/figures modules (matplotlib is absent), pins BLAS to one thread as the reference's own
`pkg/tests/conftest.py:5-9` does, and writes compressed ``.npz`` fixtures next to this script.
Nothing at test / bench time reads `/root/reference`; only these fixtures travel.

Fixtures
  shapes.npz      reference_shapes(2|3) tables and contracted Mref/sref/tref   (assembly.py:115-190,236)
  meshes.npz      reference-built meshes + promoted numbering (mesh.py:241-315, structured.py)
  c1.npz          BASELINE config 1: pattern, values, rhs, solved fields (tol 1e-10), reconstruct,
                  fixed-budget GMRES history                                    (assembly.py:403, krylov.py:63,
                                                                                 spectral.py:254-317)
  pipe3d.npz      down-scaled 3D pipe (pipe_grid(3,15)), parabolic Dirichlet inlet, modes 1 and 16
  c2_pattern.npz  BASELINE config 2 (jittered 199 800-tet pipe): pattern hash, sampled A@x and rhs
  small3d.npz     down-scaled instances of the config 3/4/5 generators (bend, Y-junction, jittered
                  pipe), two modes each solved by the reference to 1e-10
  snap.npz        field snapshots written by the reference (native text + legacy VTK, 2D and 3D)
                  as raw bytes, with their inputs                              (io.py:88-183)
  c2_gmres.npz    BASELINE config 2 fixed-budget GMRES (modes 1, 16; restart 200, 200 iterations,
                  x0 = 0): residual history, x at sampled rows, ||x|| and projections of x on
                  seeded vectors                                                 (krylov.py:63-164)
  c3_gmres.npz    BASELINE config 3 at full size (2 059 200-tet bend, n = 8.39 M): fixed-budget GMRES
                  (mode 1, restart 40, 40 iterations, x0 = 0): history, sampled x, projections
  adaptive.npz    adaptive_mode_refinement on seeded sampled waveforms: final N_m, converged flag,
                  per-mode energies and iteration counts                       (spectral.py:333-371)
  post.npz        post-processing on seeded complex fields: interpolate_at_quadrature, l2_norm,
                  field_error vs an analytic point oracle, flow_rate and patch_area of every
                  boundary patch, fit_loglog_slope             (assembly.py:497-511, metrics.py:12-113)
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
from multiprocessing import Pool
from pathlib import Path

os.environ["OMP_NUM_THREADS"] = "1"
os.environ["OPENBLAS_NUM_THREADS"] = "1"
os.environ["MKL_NUM_THREADS"] = "1"
os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

from spectralstokes import assembly as RA  # noqa: E402
from spectralstokes import krylov as RK  # noqa: E402
from spectralstokes import io as RIO  # noqa: E402
from spectralstokes import metrics as RME  # noqa: E402
from spectralstokes import mesh as RM  # noqa: E402
from spectralstokes import spectral as RSP  # noqa: E402
from spectralstokes import structured as RS  # noqa: E402

from paper_2009_06725_b200.workloads import (  # noqa: E402
    C1_TOL, c1_case, c2_case, c3_small, c4_small, c5_small, pipe3d_case,
)


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _ref_qmesh(mesh_mine, geom_kind=None, radius=None):
    """Rebuild a mesh with the REFERENCE classes and promote it with the reference."""
    patches = {n: RM.BoundaryPatch(kind=p.kind, faces=np.asarray(p.faces)) for n, p in mesh_mine.boundary_patches.items()}
    rmesh = RM.Mesh(np.asarray(mesh_mine.nodes), np.asarray(mesh_mine.elements), patches)
    geom = None
    if geom_kind == "cylinder":
        geom = RM.BoundaryGeometry(surfaces={"wall": RM.CylinderBoundary(point=(0.0, 0.0, 0.0), axis=(0.0, 0.0, 1.0), radius=radius)})
    return RM.promote_to_quadratic(rmesh, geom)


def _mesh_arrays(prefix, q):
    out = {f"{prefix}_nodes": q.nodes, f"{prefix}_elements": q.elements, f"{prefix}_vel_conn": q.vel_conn,
           f"{prefix}_edges": q.edges, f"{prefix}_nvert": np.int64(q.n_vertices)}
    names = sorted(q.boundary_patches)
    out[f"{prefix}_patch_names"] = np.array(names)
    for n in names:
        p = q.boundary_patches[n]
        out[f"{prefix}_patch_{n}_kind"] = np.array(p.kind)
        out[f"{prefix}_patch_{n}_faces"] = p.faces
        out[f"{prefix}_patch_{n}_face_conn"] = p.face_conn
    return out


def make_shapes():
    out = {}
    for dim in (2, 3):
        s = RA.reference_shapes(dim)
        out[f"d{dim}_points"] = s.points
        out[f"d{dim}_weights"] = s.weights
        out[f"d{dim}_vel_values"] = s.vel_values
        out[f"d{dim}_vel_grads"] = s.vel_grads
        out[f"d{dim}_pres_values"] = s.pres_values
        out[f"d{dim}_mref"] = np.einsum("q,qa,qb->ab", s.weights, s.vel_values, s.vel_values)
        out[f"d{dim}_sref"] = np.einsum("q,qam,qbn->abmn", s.weights, s.vel_grads, s.vel_grads)
        out[f"d{dim}_tref"] = np.einsum("q,qam,qb->amb", s.weights, s.vel_grads, s.pres_values)
    np.savez_compressed(HERE / "shapes.npz", **out)


def make_meshes():
    out = {}
    for name, (nx, ny, L, H) in {"chan10x4": (10, 4, 4.0, 1.0), "chan3x2": (3, 2, 2.0, 1.0)}.items():
        q = RM.promote_to_quadratic(RS.channel_grid(nx, ny, L, H))
        out.update(_mesh_arrays(name, q))
    for name, (nr, nl) in {"pipe2x3": (2, 3), "pipe3x4": (3, 4)}.items():
        m, g = RS.pipe_grid(nr, nl, 0.5, 5.0)
        out.update(_mesh_arrays(name, RM.promote_to_quadratic(m, g)))
    np.savez_compressed(HERE / "meshes.npz", **out)


# -- config 1 ------------------------------------------------------------------------------------

def _c1_setup():
    case = c1_case()
    q = _ref_qmesh(case.mesh)
    props = RA.FluidProps(density=case.density, viscosity=case.viscosity)
    wf = RSP.BoundaryWaveform(patch="inlet", kind="neumann", direction=np.array([1.0, 0.0]),
                              period=case.period, coefficients=case.coefficients)
    ms = RSP.fourier_transform_bcs([wf], case.n_modes)
    return case, q, props, ms


def _c1_solve(idx):
    case, q, props, ms = _c1_setup()
    t0 = time.perf_counter()
    sol = RSP._solve_one_mode(q, props, ms, RK.SolverSettings(tolerance=C1_TOL, restart=200), idx, "full")
    return idx, sol.velocity, sol.pressure, sol.report.iterations, sol.report.residual, sol.report.converged, time.perf_counter() - t0


def make_c1(pool):
    case, q, props, ms = _c1_setup()
    out = _mesh_arrays("mesh", q)
    out["coefficients"] = case.coefficients
    out["omegas"] = ms.frequencies
    patterns = []
    for i, om in enumerate(ms.frequencies):
        s = RA.assemble_mode_system(q, props, float(om), h_mode={"inlet": ms.coefficients["inlet"][i] * np.array([1.0, 0.0])})
        patterns.append((s.matrix.indptr.copy(), s.matrix.indices.copy()))
        out[f"rhs_{i}"] = s.rhs
        if i == 1:
            out["indptr"], out["indices"] = s.matrix.indptr, s.matrix.indices
            out["data_1"] = s.matrix.data
            out["vel_dof"], out["pres_dof"] = s.vel_dof, s.pres_dof
            out["jacobi_1"] = RK.jacobi_precondition(s)
            rng = np.random.default_rng(1234)
            x = rng.normal(size=s.n_dofs) + 1j * rng.normal(size=s.n_dofs)
            out["spmv_x"], out["spmv_y"] = x, s.matrix @ x
            xb, it, hist, conv = RK.gmres(s.matrix, s.rhs, tol=C1_TOL, restart=200, maxiter=200, scale=RK.jacobi_precondition(s))
            out["budget_x"], out["budget_hist"] = xb, np.array(hist)
            xb, it, hist, conv = RK.gmres(s.matrix, s.rhs, tol=C1_TOL, restart=40, maxiter=100, scale=RK.jacobi_precondition(s))
            out["budget40_x"], out["budget40_hist"] = xb, np.array(hist)
    out["pattern_same_all_omega"] = np.bool_(all(np.array_equal(a[0], patterns[0][0]) and np.array_equal(a[1], patterns[0][1]) for a in patterns))
    res = sorted(pool.map(_c1_solve, range(case.n_modes + 1)))
    sols = []
    for idx, u, p, it, r, conv, wall in res:
        out[f"u_{idx}"], out[f"p_{idx}"] = u, p
        out[f"iters_{idx}"], out[f"res_{idx}"], out[f"conv_{idx}"], out[f"wall_{idx}"] = it, r, conv, wall
        sols.append(RSP.ModeSolution(index=idx, omega=float(ms.frequencies[idx]), velocity=u, pressure=p,
                                     report=RK.SolveReport(iterations=it, residual=r, converged=conv, wall_time=wall)))
    ts = np.array([0, 5, 13, 27]) / 32.0
    out["recon_t"] = ts
    for j, t in enumerate(ts):
        out[f"recon_u_{j}"], out[f"recon_p_{j}"] = RSP.reconstruct(sols, float(t))
    np.savez_compressed(HERE / "c1.npz", **out)
    print("c1 iterations", [r[3] for r in res], "wall", sum(r[6] for r in res))


# -- down-scaled 3D pipe ---------------------------------------------------------------------------

def _pipe_solve(idx):
    case = pipe3d_case()
    q = _ref_qmesh(case.mesh, "cylinder", case.radius)
    props = RA.FluidProps(density=case.density, viscosity=case.viscosity)
    g = case.coefficients[idx] * case.profile
    s = RA.assemble_mode_system(q, props, float(case.omegas[idx]), g_mode=g)
    t0 = time.perf_counter()
    x, rep = RK.gmres_solve(s, RK.SolverSettings(tolerance=C1_TOL, restart=200))
    u, p = s.expand(x)
    return idx, u, p, rep.iterations, rep.residual, rep.converged, time.perf_counter() - t0, s


def make_pipe3d(pool):
    case = pipe3d_case()
    q = _ref_qmesh(case.mesh, "cylinder", case.radius)
    out = _mesh_arrays("mesh", q)
    out["profile"], out["coefficients"], out["omegas"] = case.profile, case.coefficients, case.omegas
    picks = [1, 16]
    res = pool.map(_pipe_solve, picks)
    for idx, u, p, it, r, conv, wall, s in res:
        out[f"u_{idx}"], out[f"p_{idx}"] = u, p
        out[f"iters_{idx}"], out[f"res_{idx}"], out[f"conv_{idx}"], out[f"wall_{idx}"] = it, r, conv, wall
        out[f"rhs_{idx}"] = s.rhs
        out[f"pattern_sha_{idx}"] = np.array(_sha(s.matrix.indptr, s.matrix.indices))
        out[f"nnz_{idx}"] = np.int64(s.matrix.nnz)
    np.savez_compressed(HERE / "pipe3d.npz", **out)
    print("pipe3d iterations", [(r[0], r[3]) for r in res])


# -- down-scaled configs 3, 4, 5 -----------------------------------------------------------------

SMALL = {"c3": (c3_small, [1, 8]), "c4": (c4_small, [1, 8]), "c5": (c5_small, [1, 16])}


def _small_solve(args):
    tag, idx = args
    case = SMALL[tag][0]()
    geom = "cylinder" if case.geometry is not None else None
    q = _ref_qmesh(case.mesh, geom, case.radius)
    props = RA.FluidProps(density=case.density, viscosity=case.viscosity)
    s = RA.assemble_mode_system(q, props, float(case.omegas[idx]), g_mode=case.coefficients[idx] * case.profile)
    t0 = time.perf_counter()
    x, rep = RK.gmres_solve(s, RK.SolverSettings(tolerance=C1_TOL, restart=200))
    u, p = s.expand(x)
    return (tag, idx, u, p, rep.iterations, rep.residual, rep.converged, time.perf_counter() - t0, s.rhs,
            _sha(s.matrix.indptr, s.matrix.indices), s.matrix.nnz, _sha(q.nodes), _sha(q.vel_conn))


def make_small3d(pool):
    jobs = [(tag, i) for tag, (_, idxs) in SMALL.items() for i in idxs]
    out = {}
    for tag, idx, u, p, it, r, conv, wall, rhs, psha, nnz, nsha, csha in pool.map(_small_solve, jobs):
        k = f"{tag}_{idx}"
        out[f"{k}_u"], out[f"{k}_p"], out[f"{k}_rhs"] = u, p, rhs
        out[f"{k}_iters"], out[f"{k}_res"], out[f"{k}_conv"], out[f"{k}_wall"] = it, r, conv, wall
        out[f"{k}_pattern_sha"], out[f"{k}_nnz"] = np.array(psha), np.int64(nnz)
        out[f"{tag}_nodes_sha"], out[f"{tag}_conn_sha"] = np.array(nsha), np.array(csha)
        print(k, it, r, conv, round(wall, 1))
    np.savez_compressed(HERE / "small3d.npz", **out)


# -- config 2 pattern --------------------------------------------------------------------------------

def make_c2_pattern():
    case = c2_case()
    t0 = time.perf_counter()
    q = _ref_qmesh(case.mesh, "cylinder", case.radius)
    props = RA.FluidProps(density=case.density, viscosity=case.viscosity)
    out = {"mesh_nodes_sha": np.array(_sha(q.nodes)), "mesh_conn_sha": np.array(_sha(q.vel_conn))}
    rng = np.random.default_rng(99)
    for idx in (0, 1):
        g = case.coefficients[idx] * case.profile
        s = RA.assemble_mode_system(q, props, float(case.omegas[idx]), g_mode=g)
        out[f"pattern_sha_{idx}"] = np.array(_sha(s.matrix.indptr, s.matrix.indices))
        out[f"nnz_{idx}"] = np.int64(s.matrix.nnz)
        out["n"] = np.int64(s.n_dofs)
        x = rng.normal(size=s.n_dofs) + 1j * rng.normal(size=s.n_dofs)
        y = s.matrix @ x
        rows = np.sort(np.random.default_rng(7).choice(s.n_dofs, 2000, replace=False))
        out[f"spmv_seed_{idx}"] = np.int64(99)
        out[f"spmv_rows_{idx}"], out[f"spmv_y_{idx}"], out[f"spmv_norm_{idx}"] = rows, y[rows], np.linalg.norm(y)
        out[f"rhs_rows_{idx}"], out[f"rhs_norm_{idx}"] = s.rhs[rows], np.linalg.norm(s.rhs)
        out[f"diag_rows_{idx}"] = s.matrix.diagonal()[rows]
        rng = np.random.default_rng(99)
    np.savez_compressed(HERE / "c2_pattern.npz", **out)
    print("c2 pattern", time.perf_counter() - t0, "s")


# -- config 2 fixed-budget GMRES (x and history after 200 iterations) ---------------

C2_GMRES_MODES = (1, 16)
C2_GMRES_SAMPLE = 20000


def _c2_gmres(idx):
    case = c2_case()
    q = _ref_qmesh(case.mesh, "cylinder", case.radius)
    props = RA.FluidProps(density=case.density, viscosity=case.viscosity)
    s = RA.assemble_mode_system(q, props, float(case.omegas[idx]), g_mode=case.coefficients[idx] * case.profile)
    sc = RK.jacobi_precondition(s)
    t0 = time.perf_counter()
    x, it, hist, conv = RK.gmres(s.matrix, s.rhs, tol=1e-10, restart=200, maxiter=200, scale=sc)
    wall = time.perf_counter() - t0
    n = s.n_dofs
    rows = np.sort(np.random.default_rng(1000 + idx).choice(n, C2_GMRES_SAMPLE, replace=False))
    rng = np.random.default_rng(2000 + idx)
    proj = np.stack([rng.normal(size=n) + 1j * rng.normal(size=n) for _ in range(4)]) @ x
    return idx, dict(hist=np.array(hist), iters=np.int64(it), conv=np.bool_(conv), rows=rows, x_rows=x[rows],
                     x_norm=np.float64(np.linalg.norm(x)), proj=proj, n=np.int64(n), wall=np.float64(wall),
                     res=np.float64(np.linalg.norm(s.rhs - s.matrix @ x) / np.linalg.norm(s.rhs)))


def make_c2_gmres(pool):
    out = {}
    for idx, d in pool.map(_c2_gmres, C2_GMRES_MODES):
        for k, v in d.items():
            out[f"{k}_{idx}"] = v
        print("c2 gmres mode", idx, "iters", int(d["iters"]), "wall", float(d["wall"]), "res", float(d["res"]))
    np.savez_compressed(HERE / "c2_gmres.npz", **out)


def make_c3_gmres():
    from paper_2009_06725_b200.workloads import c3_case

    case = c3_case()
    t0 = time.perf_counter()
    q = _ref_qmesh(case.mesh)
    props = RA.FluidProps(density=case.density, viscosity=case.viscosity)
    s = RA.assemble_mode_system(q, props, float(case.omegas[1]), g_mode=case.coefficients[1] * case.profile)
    t_asm = time.perf_counter() - t0
    sc = RK.jacobi_precondition(s)
    t0 = time.perf_counter()
    x, it, hist, conv = RK.gmres(s.matrix, s.rhs, tol=1e-10, restart=40, maxiter=40, scale=sc)
    wall = time.perf_counter() - t0
    n = s.n_dofs
    rows = np.sort(np.random.default_rng(1301).choice(n, 20000, replace=False))
    rng = np.random.default_rng(2301)
    proj = np.stack([rng.normal(size=n) + 1j * rng.normal(size=n) for _ in range(2)]) @ x
    np.savez_compressed(HERE / "c3_gmres.npz", hist=np.array(hist), iters=np.int64(it), rows=rows, x_rows=x[rows],
                        x_norm=np.float64(np.linalg.norm(x)), proj=proj, n=np.int64(n),
                        pattern_sha=np.array(_sha(s.matrix.indptr, s.matrix.indices)), nnz=np.int64(s.matrix.nnz),
                        wall=np.float64(wall), t_assembly=np.float64(t_asm))
    print("c3 gmres", it, "iterations", round(wall, 1), "s; assembly", round(t_asm, 1), "s; n", n)


# -- adaptive mode refinement (spectral.py:333-371) -------------------------------------------------

ADAPTIVE_CASES = {
    # name: (signal, period, kind, tol, max_modes)   -> reference outcome (final N_m, converged, solved)
    "square": ("square", 10.0, "neumann", 1e-3, 12),    # stops at the zero even harmonic: (1, True, 3)
    "saw": ("saw", 1.0, "neumann", 1e-2, 20),            # (11, True, 12)
    "saw_cap": ("saw", 1.0, "neumann", 2e-3, 16),        # hits max_modes: (16, False, 17)
    "noisy": ("noisy", 10.0, "neumann", 1e-2, 16),       # (8, True, 9)
}


def adaptive_signal(kind, n=128):
    """Seeded sampled signals for the adaptive fixture (tests/test_gpu_postprocess.py rebuilds them)."""
    t = np.arange(n) / n
    if kind == "square":
        return np.where(t < 0.5, 1.0, -1.0)
    if kind == "saw":
        return t - 0.5
    rng = np.random.default_rng(333)
    return np.sin(2 * np.pi * t) + 0.3 * np.sin(6 * np.pi * t + 0.4) + 0.2 * rng.normal(size=n)


def make_adaptive():
    out = {}
    q = RM.promote_to_quadratic(RS.channel_grid(6, 3, length=2.0, half_height=1.0))
    props = RA.FluidProps(density=1.0, viscosity=1.0)
    for name, (sig, period, kind, tol, mm) in ADAPTIVE_CASES.items():
        wf = RSP.BoundaryWaveform(patch="inlet", kind=kind, direction=np.array([1.0, 0.0]), period=period,
                                  samples=adaptive_signal(sig))
        sols, final_nm, conv = RSP.adaptive_mode_refinement(q, props, [wf], tol,
                                                            RK.SolverSettings(tolerance=1e-10), max_modes=mm)
        out[f"{name}_final_nm"], out[f"{name}_converged"] = np.int64(final_nm), np.bool_(conv)
        out[f"{name}_n_solved"] = np.int64(len(sols))
        out[f"{name}_energies"] = RSP.mode_energies(sols, q, period)
        out[f"{name}_iters"] = np.array([s.report.iterations for s in sols])
        out[f"{name}_u_last"] = sols[-1].velocity
        print("adaptive", name, final_nm, conv, len(sols))
    np.savez_compressed(HERE / "adaptive.npz", **out)


def post_oracle(xy):
    """Analytic point field for field_error (shared with tests/test_*_post.py): complex, dim-vector."""
    x = np.asarray(xy, dtype=float)
    d = x.shape[1]
    cols = [np.sin(1.3 * x[:, 0]) + 0.5j * x[:, 1] ** 2, np.cos(0.7 * x[:, 1]) - 0.25j * x[:, 0]]
    if d == 3:
        cols.append(x[:, 2] * x[:, 0] + 1j * np.sin(x[:, 2]))
    return np.stack(cols, axis=1)


def make_post():
    out = {}
    rng = np.random.default_rng(404)
    for name, q in (("c1", _ref_qmesh(c1_case().mesh)),
                    ("pipe3d", _ref_qmesh(pipe3d_case().mesh, "cylinder", pipe3d_case().radius))):
        out.update(_mesh_arrays(name, q))
        nvn, dim = q.n_velocity_nodes, q.dim
        vec = rng.standard_normal((nvn, dim)) + 1j * rng.standard_normal((nvn, dim))
        sca = rng.standard_normal(nvn)
        # nodal interpolant of the analytic field (so field_error is small but non-zero)
        near = post_oracle(q.nodes) + 1e-3 * vec
        out[f"{name}_vec"], out[f"{name}_sca"], out[f"{name}_near"] = vec, sca, near
        coords, vals, w = RA.interpolate_at_quadrature(q, vec)
        out[f"{name}_iq_coords"], out[f"{name}_iq_vals"], out[f"{name}_iq_w"] = coords, vals, w
        _, svals, _ = RA.interpolate_at_quadrature(q, sca)
        out[f"{name}_iq_svals"] = svals
        out[f"{name}_l2_vec"] = np.float64(RME.l2_norm(vec, q))
        out[f"{name}_field_error"] = np.float64(RME.field_error(near, post_oracle, q))
        for pn in sorted(q.boundary_patches):
            if not q.boundary_patches[pn].faces.size:
                continue
            out[f"{name}_flow_{pn}"] = np.complex128(RME.flow_rate(vec, q, pn))
            out[f"{name}_flowreal_{pn}"] = np.float64(RME.flow_rate(vec.real, q, pn))
            out[f"{name}_area_{pn}"] = np.float64(RME.patch_area(q, pn))
    xs = np.array([0.5, 0.25, 0.125, 0.0625])
    ys = 3.0 * xs ** 2.1 * (1 + 0.01 * np.array([1, -1, 1, -1]))
    out["fit_x"], out["fit_y"], out["fit_slope"] = xs, ys, np.float64(RME.fit_loglog_slope(xs, ys))
    np.savez_compressed(HERE / "post.npz", **out)
    print("post", {k: v for k, v in out.items() if "flow" in k or "area" in k or "error" in k})


def make_snapshots():
    import tempfile

    out = {}
    rng = np.random.default_rng(77)
    meshes = {"chan": _ref_qmesh(RS.channel_grid(3, 2, 2.0, 1.0))}
    m3, geom = RS.pipe_grid(2, 3, 0.5, 5.0)
    meshes["pipe"] = RM.promote_to_quadratic(m3, geom)
    with tempfile.TemporaryDirectory() as td:
        for name, q in meshes.items():
            out.update(_mesh_arrays(name, q))
            vel = rng.normal(size=(q.n_velocity_nodes, q.dim)) * 10.0 ** rng.integers(-8, 8, size=(q.n_velocity_nodes, q.dim))
            pres = rng.normal(size=q.n_vertices)
            pres[0] = 0.0
            if q.n_vertices > 2:
                pres[1], pres[2] = -0.0, 1e-310          # signed zero, subnormal
            out[f"{name}_vel"], out[f"{name}_pres"] = vel, pres
            for fmt in ("native", "vtk"):
                path = os.path.join(td, f"{name}.{fmt}")
                RIO.write_field_snapshot(path, q, vel, pres, fmt=fmt, time=0.375)
                out[f"{name}_{fmt}_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
            path = os.path.join(td, f"{name}_geom.vtk")
            RIO.write_vtk_snapshot(path, q, title="geometry only")
            out[f"{name}_vtkgeom_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
    np.savez_compressed(HERE / "snap.npz", **out)
    print("snapshots", {k: v.size for k, v in out.items() if k.endswith("_bytes")})


if __name__ == "__main__":
    what = sys.argv[1:] or ["shapes", "meshes", "c2", "c1", "pipe3d", "small3d", "post", "snap", "c2gmres",
                            "adaptive"]
    with Pool(min(9, os.cpu_count() or 1)) as pool:
        if "shapes" in what:
            make_shapes()
        if "meshes" in what:
            make_meshes()
        if "c2" in what:
            make_c2_pattern()
        if "c1" in what:
            make_c1(pool)
        if "pipe3d" in what:
            make_pipe3d(pool)
        if "small3d" in what:
            make_small3d(pool)
        if "post" in what:
            make_post()
        if "snap" in what:
            make_snapshots()
        if "c2gmres" in what:
            make_c2_gmres(pool)
        if "adaptive" in what:
            make_adaptive()
        if "c3gmres" in what:
            make_c3_gmres()
