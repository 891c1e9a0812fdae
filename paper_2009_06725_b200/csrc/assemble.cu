// Device element assembly, value export, per-mode right-hand sides, expansion and the
// standalone mode-batched SpMV.
//
// Element assembly restates assemble_{mass,stiffness}_scalar / assemble_divergence
// (reference assembly.py:151-246): per element |det J|, J^-1, then
//   M'_ab = (rho |J|) Mref_ab,  S'_ab = (mu |J|) sum_mn sref_abmn (J^-1 J^-T)_mn,
//   D_(a,d),p = -|J| sum_m tref_amp J^-1_md,
// scattered through the precomputed element->slot map, one colour per launch (elements of a
// colour share no vertex, so no two threads touch the same slot: atomic-free and deterministic).
// It runs ONCE per mesh; the reference re-assembles per mode (spectral.py:280).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "ss_common.h"
#include "ss_pattern.h"
#include "ss_spmv.cuh"

__constant__ double c_mref[100];
__constant__ double c_sref[900];
__constant__ double c_tref[120];

// ------------------------------------------------------------------------------------------------
// Reference tables (restates assembly.py:51-128 and the contractions at 169, 182, 236).
// ------------------------------------------------------------------------------------------------
static void reference_tables(int dim, std::vector<double>& mref, std::vector<double>& sref,
                             std::vector<double>& tref) {
  std::vector<std::vector<double>> bary;
  std::vector<double> w;
  if (dim == 2) {
    const double A[2] = {0.445948490915965, 0.091576213509771};
    const double W[2] = {0.223381589678011, 0.109951743655322};
    for (int g = 0; g < 2; ++g)
      for (int i = 0; i < 3; ++i) {
        std::vector<double> b(3, A[g]);
        b[i] = 1 - 2 * A[g];
        bary.push_back(b);
        w.push_back(0.5 * W[g]);
      }
  } else {
    const double s = std::sqrt(5.0 / 14.0), hi = (1.0 + s) / 4.0, lo = (1.0 - s) / 4.0;
    bary.push_back({0.25, 0.25, 0.25, 0.25});
    w.push_back(-74.0 / 5625.0);
    for (int i = 0; i < 4; ++i) {
      std::vector<double> b(4, 1.0 / 14.0);
      b[i] = 11.0 / 14.0;
      bary.push_back(b);
      w.push_back(343.0 / 45000.0);
    }
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j) {
        std::vector<double> b(4, lo);
        b[i] = hi;
        b[j] = hi;
        bary.push_back(b);
        w.push_back(56.0 / 2250.0);
      }
  }
  const int nq = (int)w.size(), nv = dim == 2 ? 6 : 10, np = dim + 1;
  const int E2[3][2] = {{0, 1}, {1, 2}, {2, 0}};
  const int E3[6][2] = {{0, 1}, {1, 2}, {0, 2}, {0, 3}, {1, 3}, {2, 3}};
  std::vector<double> val(nq * nv), grad(nq * nv * dim), lam(nq * np);
  for (int q = 0; q < nq; ++q) {
    // points = barycentric coordinates 1..dim; lambda_0 recomputed as 1 - sum (assembly.py:89-91)
    double sum = 0;
    for (int c = 1; c <= dim; ++c) sum += bary[q][c];
    double L[4];
    L[0] = 1.0 - sum;
    for (int c = 1; c <= dim; ++c) L[c] = bary[q][c];
    for (int v = 0; v < np; ++v) lam[q * np + v] = L[v];
    auto dl = [&](int v, int m) { return v == 0 ? -1.0 : (m == v - 1 ? 1.0 : 0.0); };
    for (int v = 0; v < np; ++v) {
      val[q * nv + v] = L[v] * (2.0 * L[v] - 1.0);
      for (int m = 0; m < dim; ++m) grad[(q * nv + v) * dim + m] = (4.0 * L[v] - 1.0) * dl(v, m);
    }
    for (int e = 0; e < nv - np; ++e) {
      const int i = dim == 2 ? E2[e][0] : E3[e][0], j = dim == 2 ? E2[e][1] : E3[e][1];
      val[q * nv + np + e] = 4.0 * L[i] * L[j];
      for (int m = 0; m < dim; ++m)
        grad[(q * nv + np + e) * dim + m] = 4.0 * (L[i] * dl(j, m) + L[j] * dl(i, m));
    }
  }
  mref.assign(nv * nv, 0.0);
  sref.assign(nv * nv * dim * dim, 0.0);
  tref.assign(nv * dim * np, 0.0);
  for (int q = 0; q < nq; ++q)
    for (int a = 0; a < nv; ++a) {
      for (int b = 0; b < nv; ++b) {
        mref[a * nv + b] += w[q] * val[q * nv + a] * val[q * nv + b];
        for (int m = 0; m < dim; ++m)
          for (int n = 0; n < dim; ++n)
            sref[((a * nv + b) * dim + m) * dim + n] +=
                w[q] * grad[(q * nv + a) * dim + m] * grad[(q * nv + b) * dim + n];
      }
      for (int m = 0; m < dim; ++m)
        for (int b = 0; b < np; ++b)
          tref[(a * dim + m) * np + b] += w[q] * grad[(q * nv + a) * dim + m] * lam[q * np + b];
    }
}

extern "C" int ss_reference_tables(int dim, double* mref, double* sref, double* tref) {
  if (dim != 2 && dim != 3) { ss_set_error("unsupported dimension"); return SS_ERR_ARG; }
  std::vector<double> m, s, t;
  reference_tables(dim, m, s, t);
  std::copy(m.begin(), m.end(), mref);
  std::copy(s.begin(), s.end(), sref);
  std::copy(t.begin(), t.end(), tref);
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Element kernel
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void k_assemble_color(SsOperatorDev op, const int* __restrict__ conn, const int* __restrict__ emap,
                                 int emap_stride, const int* __restrict__ elems, int count,
                                 const double* __restrict__ vnodes, double rho, double mu, int* flag,
                                 double2* __restrict__ xsm, double* __restrict__ xdp, double* __restrict__ pinv) {
  constexpr int NL = DIM == 2 ? 6 : 10, NV = DIM + 1;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int e = elems[t];
  const int* c = conn + (size_t)e * NL;
  double x[NV][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[v][d] = vnodes[(size_t)c[v] * DIM + d];
  double J[DIM][DIM];  // columns are edge vectors (assembly.py:154)
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) J[i][j] = x[j + 1][i] - x[0][i];
  double det, inv[DIM][DIM];
  if (DIM == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    inv[0][0] = J[1][1] / det; inv[0][1] = -J[0][1] / det;
    inv[1][0] = -J[1][0] / det; inv[1][1] = J[0][0] / det;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double id = 1.0 / det;
    inv[0][0] = c00 * id;
    inv[1][0] = c01 * id;
    inv[2][0] = c02 * id;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) * id;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) * id;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) * id;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) * id;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) * id;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) * id;
  }
  // MeshError contract of _element_geometry (assembly.py:156-157)
  if (!(fabs(det) >= 1e-300) || !isfinite(det)) { atomicExch(flag, 1); return; }
  const double adet = fabs(det);
  double G[DIM][DIM];
#pragma unroll
  for (int m = 0; m < DIM; ++m)
#pragma unroll
    for (int n = 0; n < DIM; ++n) {
      double s = 0;
#pragma unroll
      for (int k = 0; k < DIM; ++k) s += inv[m][k] * inv[n][k];
      G[m][n] = s;
    }
  const int* mp = emap + (size_t)e * emap_stride;
  const double smu = mu * adet, srho = rho * adet;
  for (int a = 0; a < NL; ++a) {
    for (int b = 0; b < NL; ++b) {
      const int slot = __ldg(mp + a * NL + b);
      if (slot == -1) continue;
      double s = 0;
#pragma unroll
      for (int m = 0; m < DIM; ++m)
#pragma unroll
        for (int n = 0; n < DIM; ++n) s += c_sref[((a * NL + b) * DIM + m) * DIM + n] * G[m][n];
      const double sv = smu * s, mv = srho * c_mref[a * NL + b];
      double2* dst = slot >= SS_FIXED_BASE ? xsm + (slot - SS_FIXED_BASE) : slot >= 0 ? op.sm + slot : op.lsm + (-2 - slot);
      double2 cur = *dst;
      cur.x += sv;
      cur.y += mv;
      *dst = cur;
    }
  }
  const int* mvp = mp + NL * NL;
  const int* mpv = mvp + NL * NV;
  for (int a = 0; a < NL; ++a) {
    for (int p = 0; p < NV; ++p) {
      const int s_vp = __ldg(mvp + a * NV + p), s_pv = __ldg(mpv + p * NL + a);
      if (s_vp == -1 && s_pv == -1) continue;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        double s = 0;
#pragma unroll
        for (int m = 0; m < DIM; ++m) s += c_tref[(a * DIM + m) * NV + p] * inv[m][d];
        const double dv = -(adet * s);
        if (s_vp >= SS_FIXED_BASE) xdp[(size_t)(s_vp - SS_FIXED_BASE) * DIM + d] += dv;
        else if (s_vp >= 0) op.dp[(size_t)s_vp * DIM + d] += dv;
        if (s_pv >= SS_FIXED_BASE) pinv[(size_t)(s_pv - SS_FIXED_BASE) * DIM + d] += dv;
        else if (s_pv >= 0) op.dt[(size_t)s_pv * DIM + d] += dv;
        else if (s_pv <= -2) op.ldt[(size_t)(-2 - s_pv) * DIM + d] += dv;
      }
    }
  }
}

__global__ void k_gather_diag(SsOperatorDev op) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= op.nfree) return;
  const int s = op.diag_slot[r];
  op.dsm[r] = s >= 0 ? op.sm[s] : make_double2(0.0, 0.0);
}

extern "C" int ss_assemble(ss_pattern* P, const double* vertex_nodes, double density, double viscosity,
                           void* stream_) {
  if (!P || !vertex_nodes) { ss_set_error("null argument"); return SS_ERR_ARG; }
  if (!(density > 0) || !(viscosity > 0)) { ss_set_error("density and viscosity must be positive"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  SS_CUDA(cudaSetDevice(P->device));
  std::vector<double> m, s, t;
  reference_tables(P->dim, m, s, t);
  SS_CUDA(cudaMemcpyToSymbolAsync(c_mref, m.data(), m.size() * sizeof(double), 0, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyToSymbolAsync(c_sref, s.data(), s.size() * sizeof(double), 0, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyToSymbolAsync(c_tref, t.data(), t.size() * sizeof(double), 0, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyAsync(P->d_vnodes, vertex_nodes, sizeof(double) * P->nvert * P->dim, cudaMemcpyHostToDevice, st));
  const SsOperatorDev& op = P->op;
  SS_CUDA(cudaMemsetAsync(op.sm, 0, sizeof(double2) * std::max<int64_t>(1, op.nnz_n), st));
  SS_CUDA(cudaMemsetAsync(op.dp, 0, sizeof(double) * std::max<int64_t>(1, op.nnz_p * P->dim), st));
  SS_CUDA(cudaMemsetAsync(op.dt, 0, sizeof(double) * std::max<int64_t>(1, op.nnz_t * P->dim), st));
  SS_CUDA(cudaMemsetAsync(op.lsm, 0, sizeof(double2) * std::max<size_t>(1, P->lcol.size()), st));
  SS_CUDA(cudaMemsetAsync(op.ldt, 0, sizeof(double) * std::max<size_t>(1, P->ltcol.size() * P->dim), st));
  SS_CUDA(cudaMemsetAsync(P->d_flag, 0, sizeof(int), st));
  SS_CUDA(cudaMemsetAsync(P->d_xsm, 0, sizeof(double2) * std::max<size_t>(1, P->xcol.size()), st));
  SS_CUDA(cudaMemsetAsync(P->d_xdp, 0, sizeof(double) * std::max<size_t>(1, P->xpcol.size() * P->dim), st));
  SS_CUDA(cudaMemsetAsync(P->d_pinv, 0, sizeof(double) * std::max<size_t>(1, P->pincol.size() * P->dim), st));
  for (int k = 0; k < P->ncolors; ++k) {
    const int off = P->color_ptr[k], cnt = P->color_ptr[k + 1] - off;
    if (cnt == 0) continue;
    const int bs = 128, gs = (cnt + bs - 1) / bs;
    if (P->dim == 2)
      k_assemble_color<2><<<gs, bs, 0, st>>>(op, P->d_conn, P->d_emap, P->emap_stride, P->d_color_elems + off,
                                             cnt, P->d_vnodes, density, viscosity, P->d_flag, P->d_xsm, P->d_xdp, P->d_pinv);
    else
      k_assemble_color<3><<<gs, bs, 0, st>>>(op, P->d_conn, P->d_emap, P->emap_stride, P->d_color_elems + off,
                                             cnt, P->d_vnodes, density, viscosity, P->d_flag, P->d_xsm, P->d_xdp, P->d_pinv);
    SS_LAUNCH_CHECK();
  }
  k_gather_diag<<<(P->nfree + 255) / 256, 256, 0, st>>>(op);
  SS_LAUNCH_CHECK();
  int flag = 0;
  SS_CUDA(cudaMemcpyAsync(&flag, P->d_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  if (flag) { ss_set_error("degenerate element Jacobian during assembly"); return SS_ERR_MESH; }
  P->density = density;
  P->viscosity = viscosity;
  P->assembled = true;
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Value export in vector-CSR order (the reference's reduced matrix.data at frequency omega).
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void k_export_values(SsOperatorDev op, double omega, double2* __restrict__ out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= op.n) return;
  if (row < op.nfv) {
    const int r = row / DIM, d = row % DIM;
    const int n0 = op.nptr[r], n1 = op.nptr[r + 1], p0 = op.pptr[r], p1 = op.pptr[r + 1];
    int64_t pos = (int64_t)DIM * (n0 + p0) + (int64_t)d * ((n1 - n0) + (p1 - p0));
    for (int e = n0; e < n1; ++e) {
      const double2 a = op.sm[e];
      out[pos++] = make_double2(a.x, omega == 0.0 ? 0.0 : omega * a.y);
    }
    for (int e = p0; e < p1; ++e) out[pos++] = make_double2(op.dp[(size_t)e * DIM + d], 0.0);
  } else {
    const int j = row - op.nfv;
    int64_t pos = (int64_t)DIM * (op.nnz_n + op.nnz_p) + (int64_t)DIM * op.tptr[j];
    for (int e = op.tptr[j]; e < op.tptr[j + 1]; ++e)
      for (int d = 0; d < DIM; ++d) out[pos++] = make_double2(op.dt[(size_t)e * DIM + d], 0.0);
  }
}

extern "C" int ss_export_values(const ss_pattern* P, double omega, double* data_dev, void* stream_) {
  if (!P || !data_dev) { ss_set_error("null argument"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream_;
  const int n = P->op.n;
  if (P->dim == 2) k_export_values<2><<<(n + 255) / 256, 256, 0, st>>>(P->op, omega, (double2*)data_dev);
  else k_export_values<3><<<(n + 255) / 256, 256, 0, st>>>(P->op, omega, (double2*)data_dev);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Per-mode right-hand sides: rhs = load[free] - A[free, fixed] g_fixed  (assembly.py:432-478)
// load/g: [b][nvn*dim] complex (either may be null = zero); rhs: [b][ld].
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void k_rhs(SsOperatorDev op, int64_t nvn, const double* __restrict__ omegas,
                      const double2* __restrict__ load, const double2* __restrict__ g,
                      double2* __restrict__ rhs, int64_t ld) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (row >= ld) return;
  double2* out = rhs + (size_t)b * ld;
  if (row >= op.n) { out[row] = make_double2(0.0, 0.0); return; }
  const double om = omegas[b];
  const double2* gb = g ? g + (size_t)b * nvn * DIM : nullptr;
  double2 lift = make_double2(0.0, 0.0);
  double2 base = make_double2(0.0, 0.0);
  if (row < op.nfv) {
    const int r = row / DIM, d = row % DIM;
    if (load) base = load[(size_t)b * nvn * DIM + (size_t)op.free_nodes[r] * DIM + d];
    if (gb)
      for (int e = op.lptr[r]; e < op.lptr[r + 1]; ++e) {
        const double2 a = op.lsm[e];
        const double2 av = make_double2(a.x, om == 0.0 ? 0.0 : om * a.y);
        lift = cadd(lift, cmul(av, gb[(size_t)op.lcol[e] * DIM + d]));
      }
  } else if (gb) {
    const int j = row - op.nfv;
    for (int e = op.ltptr[j]; e < op.ltptr[j + 1]; ++e)
      for (int d = 0; d < DIM; ++d) {
        const double dv = op.ldt[(size_t)e * DIM + d];
        lift = cadd(lift, cmul(make_double2(dv, 0.0), gb[(size_t)op.ltcol[e] * DIM + d]));
      }
  }
  out[row] = csub(base, lift);
}

extern "C" int ss_rhs_batched(const ss_pattern* P, int nb, const double* omegas_dev, const double* load_dev,
                              const double* g_dev, double* rhs_dev, int64_t ld, void* stream_) {
  if (!P || !rhs_dev || !omegas_dev || nb <= 0 || ld < P->op.n) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream_;
  dim3 grid((unsigned)((ld + 255) / 256), nb);
  if (P->dim == 2)
    k_rhs<2><<<grid, 256, 0, st>>>(P->op, P->nvn, omegas_dev, (const double2*)load_dev, (const double2*)g_dev,
                                   (double2*)rhs_dev, ld);
  else
    k_rhs<3><<<grid, 256, 0, st>>>(P->op, P->nvn, omegas_dev, (const double2*)load_dev, (const double2*)g_dev,
                                   (double2*)rhs_dev, ld);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Expand reduced solutions to nodal fields (assembly.py:338-346).
// u: [b][nvn*dim] complex, p: [b][nvert] complex.
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void k_expand(SsOperatorDev op, int64_t nvn, int64_t nvert, const double2* __restrict__ x, int64_t ld,
                         const double2* __restrict__ g, double2* __restrict__ u, double2* __restrict__ p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  const double2* xb = x + (size_t)b * ld;
  if (i < nvn * DIM) {
    const int64_t A = i / DIM;
    const int d = (int)(i % DIM);
    const int r = op.node_rank[A];
    double2 v;
    if (r >= 0) v = xb[(size_t)r * DIM + d];
    else v = g ? g[(size_t)b * nvn * DIM + i] : make_double2(0.0, 0.0);
    u[(size_t)b * nvn * DIM + i] = v;
  }
  if (i < nvert) {
    const int j = op.vert_pdof[i];
    p[(size_t)b * nvert + i] = j >= 0 ? xb[op.nfv + j] : make_double2(0.0, 0.0);
  }
}

extern "C" int ss_expand(const ss_pattern* P, int nb, const double* x_dev, int64_t ld, const double* g_dev,
                         double* u_dev, double* p_dev, void* stream_) {
  if (!P || !x_dev || !u_dev || !p_dev || nb <= 0) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  const int64_t m = std::max<int64_t>(P->nvn * P->dim, P->nvert);
  dim3 grid((unsigned)((m + 255) / 256), nb);
  if (P->dim == 2)
    k_expand<2><<<grid, 256, 0, st>>>(P->op, P->nvn, P->nvert, (const double2*)x_dev, ld, (const double2*)g_dev,
                                      (double2*)u_dev, (double2*)p_dev);
  else
    k_expand<3><<<grid, 256, 0, st>>>(P->op, P->nvn, P->nvert, (const double2*)x_dev, ld, (const double2*)g_dev,
                                      (double2*)u_dev, (double2*)p_dev);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Jacobi scale vectors (krylov.py:49-60) for inspection / the drop-in jacobi_precondition.
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void k_jacobi(SsOperatorDev op, const double* __restrict__ omegas, double2* __restrict__ s, int64_t ld) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (row >= ld) return;
  double2 v = make_double2(1.0, 0.0);
  if (row < op.nfv) v = saddle_jacobi(op, row / DIM, omegas[b]);
  else if (row >= op.n) v = make_double2(0.0, 0.0);
  s[(size_t)b * ld + row] = v;
}

extern "C" int ss_jacobi(const ss_pattern* P, int nb, const double* omegas_dev, double* scale_dev, int64_t ld,
                         void* stream_) {
  if (!P || !scale_dev || nb <= 0 || ld < P->op.n) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  dim3 grid((unsigned)((ld + 255) / 256), nb);
  if (P->dim == 2) k_jacobi<2><<<grid, 256, 0, st>>>(P->op, omegas_dev, (double2*)scale_dev, ld);
  else k_jacobi<3><<<grid, 256, 0, st>>>(P->op, omegas_dev, (double2*)scale_dev, ld);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Standalone mode-batched SpMV: Y[b] = s_b (.) (A(w_b) X[b])   (s = 1 unless jacobi)
// One warp per node row (all dim components) or pressure row; blockIdx.y = mode.
// ------------------------------------------------------------------------------------------------
#ifdef SS_SPMV_MINB
#define SS_SPMV_BOUNDS __launch_bounds__(256, SS_SPMV_MINB)
#else
#define SS_SPMV_BOUNDS __launch_bounds__(256)
#endif
template <int DIM>
__global__ void SS_SPMV_BOUNDS k_spmv_saddle(SsOperatorDev op, int nb, const double* __restrict__ omegas,
                                                     const double2* __restrict__ X, double2* __restrict__ Y,
                                                     int64_t ld, int jacobi) {
  // one CTA = one row block for every mode: the block's matrix slice is re-read from L1
  const int blk = blockIdx.x;
  for (int b = 0; b < nb; ++b) {
    const double om = omegas[b];
    const double2* x = X + (size_t)b * ld;
    double2* y = Y + (size_t)b * ld;
    saddle_block<DIM>(op, blk, om, x, [&](int row, double2 v) {
      if (jacobi && row < op.nfv) v = cmul(saddle_jacobi(op, row / DIM, om), v);
      y[row] = v;
    });
  }
}

// The same product with the TMA-staged row-layout streamer (persistent CTAs; each staged chunk of
// the matrix is applied to all nb modes while it sits in shared memory).
template <int DIM>
__global__ void __launch_bounds__(256, 2) k_spmv_stream(SsOperatorDev op, int nb, const double* __restrict__ omegas,
                                                     const double2* __restrict__ X, double2* __restrict__ Y,
                                                     int64_t ld, int jacobi) {
  extern __shared__ __align__(128) unsigned char sring[];
  __shared__ __align__(8) uint64_t sbar[STREAM_STAGES];
  saddle_stream<DIM>(op, nb, 1, sring, sbar, [](int) { return true; }, [&](int m) { return omegas[m]; },
                     [&](int m) { return X + (size_t)m * ld; }, [&](int m, int row, double2 v) {
                       if (jacobi && row < op.nfv) v = cmul(saddle_jacobi(op, row / DIM, omegas[m]), v);
                       Y[(size_t)m * ld + row] = v;
                     });
}

extern "C" int ss_spmv_batched(const ss_pattern* P, int nb, const double* omegas_dev, const double* x_dev,
                               double* y_dev, int64_t ld, int jacobi, void* stream_) {
  if (!P || !x_dev || !y_dev || !omegas_dev || nb <= 0 || ld < P->op.n) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream_;
  static int use_stream = -1;
  if (use_stream < 0) {
    const char* e = getenv("SS_SPMV_STREAM");
    use_stream = e ? atoi(e) : 0;
  }
  if (use_stream && P->op.nchunk > 0) {
    static bool attr = false;
    if (!attr) {
      SS_CUDA(cudaFuncSetAttribute((const void*)k_spmv_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, STREAM_SMEM));
      SS_CUDA(cudaFuncSetAttribute((const void*)k_spmv_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, STREAM_SMEM));
      attr = true;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P->device);
    const unsigned grid = (unsigned)std::max(1, std::min(P->op.nchunk, 2 * sms));
    if (P->dim == 2)
      k_spmv_stream<2><<<grid, 256, STREAM_SMEM, st>>>(P->op, nb, omegas_dev, (const double2*)x_dev, (double2*)y_dev, ld, jacobi);
    else
      k_spmv_stream<3><<<grid, 256, STREAM_SMEM, st>>>(P->op, nb, omegas_dev, (const double2*)x_dev, (double2*)y_dev, ld, jacobi);
    SS_LAUNCH_CHECK();
    return SS_OK;
  }
  const unsigned grid = (unsigned)saddle_nsb_host(P->nfree, P->npf);
  if (P->dim == 2)
    k_spmv_saddle<2><<<grid, 256, 0, st>>>(P->op, nb, omegas_dev, (const double2*)x_dev, (double2*)y_dev, ld, jacobi);
  else
    k_spmv_saddle<3><<<grid, 256, 0, st>>>(P->op, nb, omegas_dev, (const double2*)x_dev, (double2*)y_dev, ld, jacobi);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// Standalone mode-interleaved batched SpMV (the GMRES tick's SpMV): X[row][nb] -> Y[b][ld].
template <int DIM>
__global__ void __launch_bounds__(256) k_spmv_interleaved(SsOperatorDev op, int nb, const double* __restrict__ omegas,
                                                          const double2* __restrict__ X, double2* __restrict__ Y,
                                                          int64_t ld, int jacobi, int split) {
  const int blk = blockIdx.x / split, sub = blockIdx.x % split;
  saddle_block_interleaved<DIM>(op, blk, sub, split, nb, nb, X, Y, ld, jacobi, [](int) { return true; },
                                [&](int m) { return omegas[m]; }, [](int) { return 1.0; });
}

extern "C" int ss_spmv_batched_interleaved(const ss_pattern* P, int nb, const double* omegas_dev, const double* x_dev,
                                           double* y_dev, int64_t ld, int jacobi, void* stream_) {
  if (!P || !x_dev || !y_dev || !omegas_dev || nb <= 0 || ld < P->op.n) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream_;
  const int nsb = saddle_nsb_host(P->nfree, P->npf);
  const int split = std::max(1, std::min(16, (8 * 148 + nsb - 1) / nsb));
  const unsigned grid = (unsigned)(nsb * split);
  if (P->dim == 2)
    k_spmv_interleaved<2><<<grid, 256, 0, st>>>(P->op, nb, omegas_dev, (const double2*)x_dev, (double2*)y_dev, ld, jacobi, split);
  else
    k_spmv_interleaved<3><<<grid, 256, 0, st>>>(P->op, nb, omegas_dev, (const double2*)x_dev, (double2*)y_dev, ld, jacobi, split);
  SS_LAUNCH_CHECK();
  return SS_OK;
}

// Algorithmic bytes of one standalone SpMV over nb modes.
extern "C" int64_t ss_spmv_bytes(const ss_pattern* P, int nb) {
  const int64_t dim = P->dim;
  const int64_t shared = 4 * (int64_t)(P->nfree + 1) * 2 + 4 * (int64_t)(P->npf + 1) +  // nptr, pptr, tptr
                         (4 + 16) * P->op.nnz_n +                                       // ncol + (S',M')
                         (4 + 8 * dim) * P->op.nnz_p + (4 + 8 * dim) * P->op.nnz_t +    // pcol+D, tcol+D^T
                         16 * (int64_t)P->nfree;                                         // diagonal
  return shared + (int64_t)nb * 32 * P->op.n;                                            // x read + y write
}

// ------------------------------------------------------------------------------------------------
// True relative residuals ||b - A(w_b) x_b|| / ||b_b|| (||A x|| when b = 0) for nb modes
// (ComplexSaddleSystem.residual_norm, assembly.py:357-362).  Per-block partials, host sum in
// fixed order -> deterministic.
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(256) k_resid_partials(SsOperatorDev op, int nb, const double* __restrict__ omegas,
                                                        const double2* __restrict__ B, const double2* __restrict__ X,
                                                        int64_t ld, double2* __restrict__ part) {
  __shared__ double red[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x % nb, blk = blockIdx.x / nb;
  const double om = omegas[b];
  const double2* x = X + (size_t)b * ld;
  const double2* rb = B + (size_t)b * ld;
  double tt = 0, bb = 0;
  saddle_block<DIM>(op, blk, om, x, [&](int row, double2 v) {
    const double2 r = rb[row];
    tt += cabs2(csub(r, v));
    bb += cabs2(r);
  });
  tt = warp_sum(tt);
  bb = warp_sum(bb);
  if (lane == 0) { red[0][warp] = tt; red[1][warp] = bb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0;
    for (int w = 0; w < 8; ++w) { s0 += red[0][w]; s1 += red[1][w]; }
    part[(size_t)b * (gridDim.x / nb) + blk] = make_double2(s0, s1);
  }
}

extern "C" int ss_residual_norms(const ss_pattern* P, int nb, const double* omegas_dev, const double* rhs_dev,
                                 const double* x_dev, int64_t ld, double* out_host, void* stream_) {
  if (!P || nb < 1 || !omegas_dev || !rhs_dev || !x_dev || !out_host || ld < P->op.n) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  const int nblk = saddle_nsb_host(P->nfree, P->npf);
  double2* part = nullptr;
  SS_CUDA(cudaMallocAsync((void**)&part, sizeof(double2) * nblk * nb, st));
  const unsigned grid = (unsigned)(nblk * nb);
  if (P->dim == 2)
    k_resid_partials<2><<<grid, 256, 0, st>>>(P->op, nb, omegas_dev, (const double2*)rhs_dev, (const double2*)x_dev, ld, part);
  else
    k_resid_partials<3><<<grid, 256, 0, st>>>(P->op, nb, omegas_dev, (const double2*)rhs_dev, (const double2*)x_dev, ld, part);
  SS_LAUNCH_CHECK();
  std::vector<double2> h((size_t)nblk * nb);
  SS_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double2) * h.size(), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaFreeAsync(part, st));
  SS_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < nb; ++b) {
    double tt = 0, bb = 0;
    for (int q = 0; q < nblk; ++q) { tt += h[(size_t)b * nblk + q].x; bb += h[(size_t)b * nblk + q].y; }
    out_host[b] = bb == 0.0 ? std::sqrt(tt) : std::sqrt(tt) / std::sqrt(bb);
  }
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Mode-batched L2(Omega) norms of nodal velocity-space fields (metrics.l2_norm, reference
// metrics.py:12-18 with interpolate_at_quadrature, assembly.py:497-511): per element |det J|, the
// field at the degree-4 quadrature points, w_q |u_q|^2 summed over components.  Per-CTA partials,
// summed on the host in fixed order (deterministic).  fields: [b][nvn][ncomp] complex.
// ------------------------------------------------------------------------------------------------
__constant__ double c_qw[16];          // quadrature weights
__constant__ double c_phi[16 * 10];    // P2 values at the quadrature points [q][a]
__constant__ double c_lam[16 * 4];     // barycentric coordinates of the quadrature points [q][v]

template <int DIM>
__global__ void __launch_bounds__(256) k_l2_partials(const int* __restrict__ conn, const double* __restrict__ vnodes,
                                                     int64_t ne, int64_t nvn, int ncomp, int nq,
                                                     const double2* __restrict__ fields, double* __restrict__ part) {
  constexpr int NL = DIM == 2 ? 6 : 10, NV = DIM + 1;
  __shared__ double red[256];
  const int b = blockIdx.y;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (e < ne) {
    const int* c = conn + e * NL;
    double x[NV][DIM];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int d = 0; d < DIM; ++d) x[v][d] = vnodes[(size_t)c[v] * DIM + d];
    double det;
    if (DIM == 2) {
      det = (x[1][0] - x[0][0]) * (x[2][1] - x[0][1]) - (x[2][0] - x[0][0]) * (x[1][1] - x[0][1]);
    } else {
      const double a0 = x[1][0] - x[0][0], a1 = x[1][1] - x[0][1], a2 = x[1][2] - x[0][2];
      const double b0 = x[2][0] - x[0][0], b1 = x[2][1] - x[0][1], b2 = x[2][2] - x[0][2];
      const double c0 = x[3][0] - x[0][0], c1 = x[3][1] - x[0][1], c2 = x[3][2] - x[0][2];
      det = a0 * (b1 * c2 - b2 * c1) - b0 * (a1 * c2 - a2 * c1) + c0 * (a1 * b2 - a2 * b1);
    }
    const double2* f = fields + (size_t)b * nvn * ncomp;
    for (int comp = 0; comp < ncomp; ++comp) {
      double2 u[NL];
#pragma unroll
      for (int a = 0; a < NL; ++a) u[a] = f[(size_t)c[a] * ncomp + comp];
      for (int q = 0; q < nq; ++q) {
        double2 v = make_double2(0.0, 0.0);
#pragma unroll
        for (int a = 0; a < NL; ++a) {
          v.x += c_phi[q * NL + a] * u[a].x;
          v.y += c_phi[q * NL + a] * u[a].y;
        }
        acc += c_qw[q] * (v.x * v.x + v.y * v.y);
      }
    }
    acc *= fabs(det);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[(size_t)b * gridDim.x + blockIdx.x] = red[0];
}

// Degree-4 element rule of reference_shapes (assembly.py:51-128, same point order), the P2 values
// at its points [q][a] and the barycentric coordinates [q][v] (assembly.py:89-91), uploaded to
// constant memory.  Returns the number of points.
static int upload_quadrature(int dim, cudaStream_t st, int* nq_out) {
  const int nl = dim == 2 ? 6 : 10;
  std::vector<std::vector<double>> bary;
  std::vector<double> w;
  if (dim == 2) {
    const double A[2] = {0.445948490915965, 0.091576213509771};
    const double W[2] = {0.223381589678011, 0.109951743655322};
    for (int g = 0; g < 2; ++g)
      for (int i = 0; i < 3; ++i) {
        std::vector<double> bb(3, A[g]);
        bb[i] = 1 - 2 * A[g];
        bary.push_back(bb);
        w.push_back(0.5 * W[g]);
      }
  } else {
    const double s = std::sqrt(5.0 / 14.0), hi = (1.0 + s) / 4.0, lo = (1.0 - s) / 4.0;
    bary.push_back({0.25, 0.25, 0.25, 0.25});
    w.push_back(-74.0 / 5625.0);
    for (int i = 0; i < 4; ++i) {
      std::vector<double> bb(4, 1.0 / 14.0);
      bb[i] = 11.0 / 14.0;
      bary.push_back(bb);
      w.push_back(343.0 / 45000.0);
    }
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j) {
        std::vector<double> bb(4, lo);
        bb[i] = hi;
        bb[j] = hi;
        bary.push_back(bb);
        w.push_back(56.0 / 2250.0);
      }
  }
  const int nq = (int)w.size();
  const int E2[3][2] = {{0, 1}, {1, 2}, {2, 0}};
  const int E3[6][2] = {{0, 1}, {1, 2}, {0, 2}, {0, 3}, {1, 3}, {2, 3}};
  std::vector<double> phi(nq * nl);
  for (int q = 0; q < nq; ++q) {
    double sum = 0;
    for (int c = 1; c <= dim; ++c) sum += bary[q][c];
    double L[4];
    L[0] = 1.0 - sum;
    for (int c = 1; c <= dim; ++c) L[c] = bary[q][c];
    for (int v = 0; v <= dim; ++v) phi[q * nl + v] = L[v] * (2.0 * L[v] - 1.0);
    for (int e = 0; e < nl - dim - 1; ++e) {
      const int i = dim == 2 ? E2[e][0] : E3[e][0], j = dim == 2 ? E2[e][1] : E3[e][1];
      phi[q * nl + dim + 1 + e] = 4.0 * L[i] * L[j];
    }
  }
  std::vector<double> lam(nq * 4, 0.0);
  for (int q = 0; q < nq; ++q) {
    double sum = 0;
    for (int c = 1; c <= dim; ++c) sum += bary[q][c];
    lam[q * 4] = 1.0 - sum;
    for (int c = 1; c <= dim; ++c) lam[q * 4 + c] = bary[q][c];
  }
  SS_CUDA(cudaMemcpyToSymbolAsync(c_qw, w.data(), sizeof(double) * nq, 0, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyToSymbolAsync(c_phi, phi.data(), sizeof(double) * nq * nl, 0, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemcpyToSymbolAsync(c_lam, lam.data(), sizeof(double) * nq * 4, 0, cudaMemcpyHostToDevice, st));
  *nq_out = nq;
  return SS_OK;
}

extern "C" int ss_l2_norms(const ss_pattern* P, int nb, int ncomp, const double* fields_dev, double* out_host,
                           void* stream_) {
  if (!P || nb < 1 || ncomp < 1 || !fields_dev || !out_host) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream_;
  const int dim = P->dim;
  int nq = 0;
  if (int rc = upload_quadrature(dim, st, &nq)) return rc;
  const int nblk = (int)((P->ne + 255) / 256);
  double* part = nullptr;
  SS_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * nblk * nb, st));
  dim3 grid(nblk, nb);
  if (dim == 2)
    k_l2_partials<2><<<grid, 256, 0, st>>>(P->d_conn, P->d_vnodes, P->ne, P->nvn, ncomp, nq, (const double2*)fields_dev, part);
  else
    k_l2_partials<3><<<grid, 256, 0, st>>>(P->d_conn, P->d_vnodes, P->ne, P->nvn, ncomp, nq, (const double2*)fields_dev, part);
  SS_LAUNCH_CHECK();
  std::vector<double> h((size_t)nblk * nb);
  SS_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaFreeAsync(part, st));
  SS_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < nb; ++b) {
    double acc = 0;
    for (int q = 0; q < nblk; ++q) acc += h[(size_t)b * nblk + q];
    out_host[b] = std::sqrt(acc);
  }
  return SS_OK;
}

// ------------------------------------------------------------------------------------------------
// Nodal velocity-space field -> values at the element quadrature points (assembly.py:497-511):
// coords[e][q][d] = sum_v lam[q][v] x_v,  vals[e][q][c] = sum_a phi[q][a] f[conn[e][a]][c],
// w[e][q] = |det J_e| * weight_q.  One thread per element.
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(256) k_interp_quad(const int* __restrict__ conn, const double* __restrict__ vnodes,
                                                     int64_t ne, int ncomp, int nq,
                                                     const double2* __restrict__ f, double* __restrict__ coords,
                                                     double2* __restrict__ vals, double* __restrict__ w) {
  constexpr int NL = DIM == 2 ? 6 : 10, NV = DIM + 1;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int* c = conn + e * NL;
  double x[NV][DIM];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[v][d] = vnodes[(size_t)c[v] * DIM + d];
  double det;
  if (DIM == 2) {
    det = (x[1][0] - x[0][0]) * (x[2][1] - x[0][1]) - (x[2][0] - x[0][0]) * (x[1][1] - x[0][1]);
  } else {
    const double a0 = x[1][0] - x[0][0], a1 = x[1][1] - x[0][1], a2 = x[1][2] - x[0][2];
    const double b0 = x[2][0] - x[0][0], b1 = x[2][1] - x[0][1], b2 = x[2][2] - x[0][2];
    const double c0 = x[3][0] - x[0][0], c1 = x[3][1] - x[0][1], c2 = x[3][2] - x[0][2];
    det = a0 * (b1 * c2 - b2 * c1) - b0 * (a1 * c2 - a2 * c1) + c0 * (a1 * b2 - a2 * b1);
  }
  for (int q = 0; q < nq; ++q) {
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double acc = 0.0;
#pragma unroll
      for (int v = 0; v < NV; ++v) acc += c_lam[q * 4 + v] * x[v][d];
      coords[((size_t)e * nq + q) * DIM + d] = acc;
    }
    w[(size_t)e * nq + q] = fabs(det) * c_qw[q];
  }
  for (int comp = 0; comp < ncomp; ++comp) {
    double2 u[NL];
#pragma unroll
    for (int a = 0; a < NL; ++a) u[a] = f[(size_t)c[a] * ncomp + comp];
    for (int q = 0; q < nq; ++q) {
      double2 v = make_double2(0.0, 0.0);
#pragma unroll
      for (int a = 0; a < NL; ++a) {
        v.x += c_phi[q * NL + a] * u[a].x;
        v.y += c_phi[q * NL + a] * u[a].y;
      }
      vals[((size_t)e * nq + q) * ncomp + comp] = v;
    }
  }
}

extern "C" int ss_quadrature_points(int dim, int* nq) {
  if ((dim != 2 && dim != 3) || !nq) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  *nq = dim == 2 ? 6 : 11;
  return SS_OK;
}

extern "C" int ss_interp_quadrature(const ss_pattern* P, int ncomp, const double* nodal_dev, double* coords_dev,
                                    double* vals_dev, double* w_dev, void* stream_) {
  if (!P || ncomp < 1 || !nodal_dev || !coords_dev || !vals_dev || !w_dev) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)stream_;
  int nq = 0;
  if (int rc = upload_quadrature(P->dim, st, &nq)) return rc;
  const unsigned grid = (unsigned)((P->ne + 255) / 256);
  if (P->dim == 2)
    k_interp_quad<2><<<grid, 256, 0, st>>>(P->d_conn, P->d_vnodes, P->ne, ncomp, nq, (const double2*)nodal_dev,
                                            coords_dev, (double2*)vals_dev, w_dev);
  else
    k_interp_quad<3><<<grid, 256, 0, st>>>(P->d_conn, P->d_vnodes, P->ne, ncomp, nq, (const double2*)nodal_dev,
                                            coords_dev, (double2*)vals_dev, w_dev);
  SS_LAUNCH_CHECK();
  return SS_OK;
}
