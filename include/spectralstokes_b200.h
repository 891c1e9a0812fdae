/*
 * spectralstokes_b200 — C ABI of the B200-native spectral-Stokes hot path (libss_b200.so).
 *
 * The reference (arXiv 2009.06725's Python package `spectralstokes`, mounted at
 * /root/reference/pkg) has no FFI: its boundary is the Python API re-exported in
 * pkg/src/spectralstokes/__init__.py:10-46.  Each entry point below replaces the reference
 * function named beside it; the Python package paper_2009_06725_b200 binds them with ctypes
 * (INTEGRATION.md shows the binding a reference maintainer would add).
 *
 * Conventions
 *   - every function returns 0 (SS_OK) or an error code; nothing throws across the ABI;
 *     ss_last_error() returns the calling thread's last message.  Codes: 1 = bad argument (ValueError),
 *     2 = mesh error (MeshError), 3 = CUDA/driver (DeviceError), 4 = misuse (RuntimeError).
 *   - complex128 arrays are interleaved {re, im} doubles;
 *   - pointers named *_dev are device pointers owned by the caller; *_host are host pointers;
 *   - stream is a cudaStream_t (NULL = legacy default stream);
 *   - per-mode vectors are mode-major with a leading dimension `ld` (complex elements).
 *   - the library owns only its opaque handles (ss_pattern, ss_krylov) and never frees caller memory.
 */
#ifndef SPECTRALSTOKES_B200_H
#define SPECTRALSTOKES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ss_pattern ss_pattern; /* mesh numbering + symbolic pattern + device operator  */
typedef struct ss_krylov ss_krylov;   /* batched GMRES workspace (basis, Hessenberg, state)   */
typedef struct ss_comm ss_comm;       /* NCCL communicator for the mode-field gather          */

#define SS_COMM_ID_BYTES 128

/* ABI revision: the Python binding refuses (rebuilds) a library whose ss_version() differs. */
#define SS_ABI_VERSION 5

const char* ss_last_error(void);
int ss_version(void);
int64_t ss_launch_count(void); /* kernels launched by this library so far (graph nodes counted) */

/* Reference tables Mref(nv x nv), sref(nv x nv x dim x dim), tref(nv x dim x (dim+1)) of the degree-4
 * rules; replaces reference_shapes + the einsum contractions (assembly.py:115-128,169,182,236). */
int ss_reference_tables(int dim, double* mref, double* sref, double* tref);

/* Symbolic reduced pattern, DOF maps, element->slot maps and element colouring.
 * Replaces the pattern half of assemble_mode_system (assembly.py:424-479: kron/bmat/COO->CSR,
 * vel_dof/pres_dof numbering at 455-475, reduction a_full[free][:, free] at 477-479).
 * vel_conn: n_elements x (6|10) int64, fixed_mask: n_vel_nodes uint8 (dirichlet/wall nodes,
 * constrained_velocity_nodes assembly.py:392-400), pinned_pressure per assembly.py:460-464. */
int ss_pattern_create(int dim, int64_t n_vel_nodes, int64_t n_vertices, int64_t n_elements,
                      const int64_t* vel_conn_host, const uint8_t* fixed_mask_host, int pinned_pressure,
                      int device, ss_pattern** out);
void ss_pattern_destroy(ss_pattern* p);
/* info[16]: n, nnz, n_free_nodes, n_free_pressures, nnz_node, nnz_vp, nnz_pv, n_colors,
 *           nnz_lift, nnz_lift_t, dim, pinned, element-map bytes, n_vel_nodes, n_vertices, n_elements */
int ss_pattern_info(const ss_pattern* p, int64_t* info);
/* Bit-exact reduced CSR pattern (= ComplexSaddleSystem.matrix.indptr/.indices, assembly.py:479).
 * indices may be NULL to obtain indptr only. */
int ss_pattern_export(const ss_pattern* p, int32_t* indptr_host, int32_t* indices_host);
/* Columns of selected rows of the same reduced CSR (sampled parity checks on very large meshes).
 * counts[i] receives the nnz of rows[i]; indices (capacity cap, may be NULL) the concatenated columns. */
int ss_pattern_export_rows(const ss_pattern* p, int64_t nrows, const int64_t* rows_host, int64_t* counts_host,
                           int32_t* indices_host, int64_t cap);
/* Constrained rows a_full[fixed_idx] at frequency omega in the unreduced numbering
 * (ComplexSaddleSystem.constrained_rows, assembly.py:471-476,491): info_out = {nrows, nnz};
 * pass NULL arrays to query sizes.  data: nnz complex. */
int ss_constrained_rows(const ss_pattern* p, double omega, int64_t* info_out, int64_t* indptr_host,
                        int32_t* indices_host, double* data_host);
/* ComplexSaddleSystem.vel_dof (n_vel_nodes x dim) and .pres_dof (n_vertices) (assembly.py:319-320). */
int ss_pattern_dof_maps(const ss_pattern* p, int64_t* vel_dof_host, int64_t* pres_dof_host);

/* Device element assembly of S' = mu*S, M' = rho*M and D once per mesh, colour by colour,
 * atomic-free.  Replaces _element_geometry + assemble_{mass,stiffness}_scalar +
 * assemble_divergence (assembly.py:151-246).  vertex_nodes_host: n_vertices x dim.
 * Returns 2 (MeshError) for a degenerate Jacobian (assembly.py:156-157). */
int ss_assemble(ss_pattern* p, const double* vertex_nodes_host, double density, double viscosity, void* stream);
/* Values of the reduced matrix at frequency omega in the exported CSR order
 * (= ComplexSaddleSystem.matrix.data, assembly.py:425-430,479).  data_dev: nnz complex. */
int ss_export_values(const ss_pattern* p, double omega, double* data_dev, void* stream);

/* Consistent traction load on a patch, accumulated into load_host (n_vel_nodes x dim complex).
 * Replaces boundary_traction_load/_surface_load (assembly.py:249-305).
 * h_kind 0: uniform (dim complex), 1: per face (n_faces x dim), 2: nodal (n_vel_nodes x dim). */
int ss_surface_load(int dim, int64_t n_vel_nodes, const double* nodes_host, int64_t n_faces,
                    const int64_t* face_conn_host, int h_kind, const double* h_host, double* load_host);
/* rhs_b = load_b[free] - A(omega_b)[free, fixed] g_b[fixed] for nb modes
 * (assembly.py:432-478).  load_dev / g_dev: nb x n_vel_nodes*dim complex (NULL = 0);
 * omegas_dev: nb doubles; rhs_dev: nb x ld complex. */
int ss_rhs_batched(const ss_pattern* p, int nb, const double* omegas_dev, const double* load_dev,
                   const double* g_dev, double* rhs_dev, int64_t ld, void* stream);
/* Mode-batched SpMV Y_b = s_b .* (A(omega_b) X_b), s = Jacobi scale if jacobi else 1.
 * Replaces `matrix @ q` / `scale * (matrix @ q)` (krylov.py:94,108,155; assembly.py:362). */
int ss_spmv_batched(const ss_pattern* p, int nb, const double* omegas_dev, const double* x_dev,
                    double* y_dev, int64_t ld, int jacobi, void* stream);
/* Same product with the mode-interleaved input layout the GMRES tick uses: x_dev is [row][nb]
 * (x[row*nb + b]), y_dev is [b][ld].  Gathers of one node return all modes' values contiguously. */
int ss_spmv_batched_interleaved(const ss_pattern* p, int nb, const double* omegas_dev, const double* x_dev,
                                double* y_dev, int64_t ld, int jacobi, void* stream);
/* Algorithmic bytes of one ss_spmv_batched call over nb modes (roofline numerator). */
int64_t ss_spmv_bytes(const ss_pattern* p, int nb);
/* True relative residuals ||b - A x||/||b|| (||A x|| if b = 0) per mode (ComplexSaddleSystem.residual_norm,
 * assembly.py:357-362).  out_host: nb doubles. */
int ss_residual_norms(const ss_pattern* p, int nb, const double* omegas_dev, const double* rhs_dev, const double* x_dev,
                      int64_t ld, double* out_host, void* stream);
/* L2(Omega) norms of nb nodal velocity-space fields (nb x n_vel_nodes x ncomp complex) by element
 * quadrature (metrics.l2_norm, metrics.py:12-18; interpolate_at_quadrature, assembly.py:497-511). */
int ss_l2_norms(const ss_pattern* p, int nb, int ncomp, const double* fields_dev, double* out_host, void* stream);
/* Points of the degree-4 element rule of reference_shapes(dim) (assembly.py:51-86): 6 (2D), 11 (3D). */
int ss_quadrature_points(int dim, int* nq);
/* Nodal velocity-space field (n_vel_nodes x ncomp complex) -> quadrature coordinates (ne x nq x dim),
 * values (ne x nq x ncomp complex) and Jacobian-weighted weights (ne x nq), all device buffers
 * (interpolate_at_quadrature, assembly.py:497-511; used by metrics.field_error, metrics.py:21-39). */
int ss_interp_quadrature(const ss_pattern* p, int ncomp, const double* nodal_dev, double* coords_dev,
                         double* vals_dev, double* w_dev, void* stream);
/* Jacobi scale vectors 1/diag (1 where diag = 0) per mode (jacobi_precondition, krylov.py:49-60). */
int ss_jacobi(const ss_pattern* p, int nb, const double* omegas_dev, double* scale_dev, int64_t ld, void* stream);
/* Reduced solutions -> nodal velocity (nb x n_vel_nodes*dim) and pressure (nb x n_vertices),
 * Dirichlet values from g_dev (ComplexSaddleSystem.expand, assembly.py:338-346). */
int ss_expand(const ss_pattern* p, int nb, const double* x_dev, int64_t ld, const double* g_dev,
              double* u_dev, double* p_dev, void* stream);

/* Batched restarted GMRES workspace on the structured operator of `p` (gmres, krylov.py:63-164). */
int ss_krylov_create_saddle(const ss_pattern* p, int max_batch, int restart, int64_t hist_cap, ss_krylov** out);
/* Same on an arbitrary complex CSR matrix (drop-in gmres(matrix, rhs, ...) for any scipy matrix).
 * vals_host: nvals x nnz complex (nvals = 1 shared or one set per mode); scale_host: optional
 * nvals x n complex left preconditioner (krylov.py:63 `scale`); jacobi_from_diag != 0 (and no
 * scale_host) computes 1/diag on the device (jacobi_precondition, krylov.py:49-60). */
int ss_krylov_create_csr(int device, int n, int64_t nnz, const int32_t* indptr_host, const int32_t* indices_host,
                         int nvals, const double* vals_host, const double* scale_host, int jacobi_from_diag,
                         int max_batch, int restart, int64_t hist_cap, ss_krylov** out);
void ss_krylov_destroy(ss_krylov* k);
/* info[10]: n, ld, restart, n_segments, segment_rows, spmv_blocks, max_batch, ticks_per_graph,
 *           pass shared-memory bytes, kind */
int ss_krylov_info(const ss_krylov* k, int64_t* info);
/* Workspace option (drops cached graphs): "row_spmv" (0/1: mode-interleaved or row-layout tick
 * SpMV; default by n), "stream_spmv" (0/1: row layout through the TMA-staged persistent kernel),
 * "device_loop" (0/1), "ticks_per_graph" (1..1024), "fused" (0/1: persistent cooperative tick),
 * "pass_alt" (0/1: basis passes stream their segments in alternating directions, for L2 reuse
 * between consecutive passes; changes the order of the passes' row sums).  Results never depend on
 * ticks_per_graph/device_loop; the SpMV layout changes no per-row summation order either. */
int ss_krylov_set_option(ss_krylov* k, const char* name, int64_t value);
/* Current value of a workspace option (names as for ss_krylov_set_option). */
int ss_krylov_get_option(const ss_krylov* k, const char* name, int64_t* value);
/* The workspace's own RHS and X buffers (nb x ld complex, device) for zero-copy callers. */
int ss_krylov_buffers(ss_krylov* k, double** rhs_dev, double** x_dev, int64_t* ld);
/* Solve nb modes to relative tolerance tol (krylov.py:63-164 semantics per mode).
 * rhs_dev/x_dev (nb x ld_in complex) may be NULL to use the workspace buffers in place;
 * use_x0 != 0 starts from x (krylov.py:79).  out_int[6*b+{iterations, converged, breakdown, phase, history length, zero rhs}],
 * out_dbl[4*b+{true residual at last cycle end, last estimate, ||b||, final target}]. */
int ss_krylov_solve(ss_krylov* k, int nb, const double* omegas_host, const int* sets_host, const double* rhs_dev,
                    double* x_dev, int64_t ld_in, int use_x0, double tol, int64_t maxiter, int jacobi,
                    void* stream, int64_t* out_int, double* out_dbl);
/* Per-iteration preconditioned residual estimates of mode b (SolveReport.residual_history). */
int ss_krylov_history(const ss_krylov* k, int mode, int64_t count, double* out_host);
/* Tick (one SpMV + three basis passes over the batch) at which each mode of the last solve
 * finished; SolveReport.wall_time of a mode = batch wall time x its tick / all ticks. */
int ss_krylov_done_ticks(const ss_krylov* k, int nb, int64_t* out_host);
/* Ticks and kernel launches of the last solve. */
int ss_krylov_last_stats(const ss_krylov* k, int64_t* ticks, int64_t* launches);
/* True relative residuals ||b - A x||/||b|| of the workspace's X (residual_norm, assembly.py:357-362). */
int ss_krylov_residuals(ss_krylov* k, int nb, void* stream, double* out_host);
/* Copy nb vectors caller <-> workspace (dir 0: buf -> RHS, 1: buf -> X, 2: X -> buf). */
int ss_krylov_copy(ss_krylov* k, int nb, int dir, double* buf_dev, int64_t ld_in, void* stream);
/* Jacobi scale (1/diag) of a CSR workspace's value set (jacobi_precondition on a matrix, krylov.py:49-60). */
int ss_krylov_csr_scale(const ss_krylov* k, int set, double* scale_host);
/* Instrumented solve (no graph; CUDA events between kernels) for the roofline: per kernel kind
 * (0 spmv, 1 c = Q^H w, 2 w -= Qc & c2 = Q^H w, 3 w -= Q c2 & ||w||, 4 x += Q y) the summed device time
 * ms_out[5], algorithmic bytes bytes_out[5] (basis passes only) and launch counts launches_out[5]. */
int ss_krylov_profile(ss_krylov* k, int nb, const double* omegas_host, double tol, int64_t maxiter, int jacobi,
                      void* stream, double* ms_out, int64_t* bytes_out, int64_t* launches_out);
/* Isolated Gram-Schmidt pass timing (which = 1: c = Q^H w; 2: fused w -= Qc, c2 = Q^H w). */
int ss_krylov_bench_pass(ss_krylov* k, int nb, int kidx, int which, int reps, void* stream, float* ms, int64_t* bytes);

/* out[t][i] = sum_b Re(fields_b[i] * phases[b][t]) for nt samples (reconstruct, spectral.py:308-317).
 * fields_dev: nb x n complex; phases_dev: nb x nt complex; out_dev: nt x n doubles. */
int ss_reconstruct(int nb, int nt, int64_t n, const double* fields_dev, const double* phases_dev, double* out_dev,
                   void* stream);

/* ---- Multi-GPU mode sharding (one process per GPU): the collective that replaces
 * the reference's in-process ModeSolution list of the thread pool (spectral.py:296-305).  NCCL is
 * dlopen'ed at first use (SS_NCCL_LIB, default "libnccl.so.2"). ---- */
/* NCCL version code of the loaded library (e.g. 22809), or -1 if NCCL cannot be loaded. */
int ss_comm_nccl_version(void);
/* ncclGetUniqueId: SS_COMM_ID_BYTES bytes made on one rank and shared out of band. */
int ss_comm_unique_id(uint8_t* id_out);
/* ncclCommInitRank on `device`. */
int ss_comm_create(int nranks, int rank, const uint8_t* id, int device, ss_comm** out);
void ss_comm_destroy(ss_comm* c);
/* Gather solved modal fields (complex128) to `root`: rank r sends its counts[r] fields (count
 * complex values each, stride ld, from send_dev); the root stores field j of rank r at
 * recv_dev + dest[counts[0] + ... + counts[r-1] + j] * ld.  One grouped ncclSend/ncclRecv round. */
int ss_comm_gather_modes(ss_comm* c, const double* send_dev, int64_t n_local, int64_t count, int64_t ld,
                         double* recv_dev, const int64_t* counts_host, const int64_t* dest_host, int root,
                         void* stream);
/* In-place sum over ranks of n doubles into the root's buffer (ncclReduce): per-GPU partial
 * reconstructions sum to u(x, t) on one rank (fused reconstruction + collective). */
int ss_comm_reduce_sum(ss_comm* c, double* buf_dev, int64_t n, int root, void* stream);
/* In-place elementwise max over ranks of n doubles on the device. */
int ss_comm_allreduce_max(ss_comm* c, double* buf_dev, int64_t n, void* stream);

/* ---- Field snapshots (host runtime, io.py:88-183): "%.17g" text, byte-identical to the reference's
 * "{:.17g}" writer, formatted/parsed in parallel.  Paths are NUL-terminated UTF-8. ---- */
/* Native snapshot (io.py:104-114).  nodes/velocity: n_vel x dim, pressure: n_vert. */
int ss_write_snapshot(const char* path, int dim, int64_t n_vel, int64_t n_vert, const double* nodes,
                      const double* velocity, const double* pressure, double time);
/* Legacy-VTK quadratic unstructured grid (write_vtk_snapshot, io.py:140-183); velocity / pressure
 * may be NULL; mid-edge pressures from edges (n_vel - n_vert x 2). */
int ss_write_vtk(const char* path, const char* title, int dim, int64_t n_vel, int64_t n_vert, const double* nodes,
                 int64_t ne, int nloc, const int64_t* vel_conn, const int64_t* edges, const double* velocity,
                 const double* pressure);
/* Data blocks of a native snapshot whose header the caller parsed (read_field_snapshot, io.py:117-134). */
int ss_read_snapshot(const char* path, int dim, int64_t n_vel, int64_t n_vert, double* coords, double* velocity,
                     double* pressure);

#ifdef __cplusplus
}
#endif
#endif
