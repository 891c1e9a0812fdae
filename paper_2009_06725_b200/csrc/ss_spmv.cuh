// Mode-batched complex SpMV building blocks for the structured saddle operator
//   A(w) = [[ S' (x) I + i w M' (x) I , D ], [ D^T, 0 ]]   (reference assembly.py:424-430)
// The node-level pattern stores one (S', M') pair per free node pair and applies it to all `dim`
// velocity components (kron structure), so the matrix stream is ~dim x smaller than the vector
// CSR; D is stored per (node, pressure) pair as `dim` doubles, once in row order (velocity rows)
// and once transposed (pressure rows).  w*M' is formed in registers per mode.
#pragma once
#include "ss_common.h"

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }

// Smith's complex division a / b (numpy's npy_cdiv algorithm).
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  const double abs_br = fabs(b.x), abs_bi = fabs(b.y);
  if (abs_br >= abs_bi) {
    if (abs_br == 0.0 && abs_bi == 0.0) return make_double2(a.x / abs_br, a.y / abs_bi);
    const double rat = b.y / b.x;
    const double scl = 1.0 / (b.x + b.y * rat);
    return make_double2((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  const double rat = b.x / b.y;
  const double scl = 1.0 / (b.y + b.x * rat);
  return make_double2((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Jacobi scale of velocity node row r at frequency w: 1/(S'_rr + i w M'_rr), 1 if that is 0
// (krylov.py:49-60 on the reduced matrix's diagonal; the pressure diagonal is 0 -> 1).
__device__ __forceinline__ double2 saddle_jacobi(const SsOperatorDev& op, int r, double omega) {
  const double2 d = op.dsm[r];
  const double2 a = make_double2(d.x, omega == 0.0 ? 0.0 : omega * d.y);
  if (a.x == 0.0 && a.y == 0.0) return make_double2(1.0, 0.0);
  return cdiv(make_double2(1.0, 0.0), a);
}

// One warp computes all DIM components of velocity node row r: acc[d] = (A x)_(r,d), result valid
// in every lane after the butterfly (lane 0's value is used; the tree is fixed -> deterministic).
template <int DIM>
__device__ __forceinline__ void saddle_vel_row(const SsOperatorDev& op, int r, double omega,
                                               const double2* __restrict__ x, int lane,
                                               double2 (&acc)[DIM]) {
#pragma unroll
  for (int d = 0; d < DIM; ++d) acc[d] = make_double2(0.0, 0.0);
  const int e0 = __ldg(op.nptr + r), e1 = __ldg(op.nptr + r + 1);
  for (int e = e0 + lane; e < e1; e += 32) {
    const int B = __ldg(op.ncol + e);
    const double2 a = __ldg(op.sm + e);
    const double am = omega * a.y;
    const double2* xb = x + (size_t)B * DIM;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const double2 v = xb[d];
      acc[d].x += a.x * v.x - am * v.y;
      acc[d].y += a.x * v.y + am * v.x;
    }
  }
  const int p0 = __ldg(op.pptr + r), p1 = __ldg(op.pptr + r + 1);
  for (int e = p0 + lane; e < p1; e += 32) {
    const double2 v = x[op.nfv + __ldg(op.pcol + e)];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const double dv = __ldg(op.dp + (size_t)e * DIM + d);
      acc[d].x += dv * v.x;
      acc[d].y += dv * v.y;
    }
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    acc[d].x = warp_sum(acc[d].x);
    acc[d].y = warp_sum(acc[d].y);
  }
}

// One warp computes pressure row j: sum over free nodes B, components d of D[(B,d),P] x_(B,d).
template <int DIM>
__device__ __forceinline__ double2 saddle_pres_row(const SsOperatorDev& op, int j,
                                                   const double2* __restrict__ x, int lane, int xs = 1) {
  double2 acc = make_double2(0.0, 0.0);
  const int e0 = __ldg(op.tptr + j), e1 = __ldg(op.tptr + j + 1);
  for (int e = e0 + lane; e < e1; e += 32) {
    const double2* xb = x + (size_t)__ldg(op.tcol + e) * DIM * xs;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const double dv = __ldg(op.dt + (size_t)e * DIM + d);
      const double2 v = xb[(size_t)d * xs];
      acc.x += dv * v.x;
      acc.y += dv * v.y;
    }
  }
  acc.x = warp_sum(acc.x);
  acc.y = warp_sum(acc.y);
  return acc;
}

// Generic complex CSR row (drop-in gmres on arbitrary matrices): warp per row.
__device__ __forceinline__ double2 csr_row(const SsCsrDev& A, int set, int row,
                                           const double2* __restrict__ x, int lane) {
  double2 acc = make_double2(0.0, 0.0);
  const double2* vals = A.vals + (size_t)set * A.nnz;
  const int e0 = __ldg(A.indptr + row), e1 = __ldg(A.indptr + row + 1);
  for (int e = e0 + lane; e < e1; e += 32) {
    const double2 a = __ldg(vals + e);
    const double2 v = x[__ldg(A.indices + e)];
    acc.x += a.x * v.x - a.y * v.y;
    acc.y += a.x * v.y + a.y * v.x;
  }
  acc.x = warp_sum(acc.x);
  acc.y = warp_sum(acc.y);
  return acc;
}

// ------------------------------------------------------------------------------------------------
// Block-row SpMV iterator shared by every SpMV-shaped kernel (standalone, GMRES tick, residuals).
// A CTA of 256 threads owns a fixed block of rows of ONE mode (block -> rows never depends on the
// batch, so per-mode reductions are batch-invariant):
//   velocity blocks: 128 free velocity NODE rows, 8 lanes per node row (all dim components);
//   pressure blocks: 32 pressure rows, one warp per row.
// emit(row, value) is called by exactly one lane per output row.
// ------------------------------------------------------------------------------------------------
constexpr int SPMV_VROWS = 128;   // node rows per velocity block
constexpr int SPMV_PROWS = 32;    // pressure (or generic CSR) rows per block

__device__ __forceinline__ int saddle_nvb(const SsOperatorDev& op) { return (op.nfree + SPMV_VROWS - 1) / SPMV_VROWS; }
__device__ __host__ __forceinline__ int saddle_nsb_host(int nfree, int npf) {
  return (nfree + SPMV_VROWS - 1) / SPMV_VROWS + (npf + SPMV_PROWS - 1) / SPMV_PROWS;
}

template <int DIM>
__device__ __forceinline__ void saddle_vel_row_g8(const SsOperatorDev& op, int r, double omega,
                                                  const double2* __restrict__ x, int gl, double2 (&acc)[DIM],
                                                  int xs = 1) {
#pragma unroll
  for (int d = 0; d < DIM; ++d) acc[d] = make_double2(0.0, 0.0);
  if (r >= 0) {
    const int e0 = __ldg(op.nptr + r), e1 = __ldg(op.nptr + r + 1);
#pragma unroll 4
    for (int e = e0 + gl; e < e1; e += 8) {
      const int B = __ldg(op.ncol + e);
      const double2 a = __ldg(op.sm + e);
      const double am = omega * a.y;
      const double2* xb = x + (size_t)B * DIM * xs;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double2 v = xb[(size_t)d * xs];
        acc[d].x += a.x * v.x - am * v.y;
        acc[d].y += a.x * v.y + am * v.x;
      }
    }
    const int p0 = __ldg(op.pptr + r), p1 = __ldg(op.pptr + r + 1);
#pragma unroll 2
    for (int e = p0 + gl; e < p1; e += 8) {
      const double2 v = x[(size_t)(op.nfv + __ldg(op.pcol + e)) * xs];
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double dv = __ldg(op.dp + (size_t)e * DIM + d);
        acc[d].x += dv * v.x;
        acc[d].y += dv * v.y;
      }
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      acc[d].x += __shfl_xor_sync(0xffffffffu, acc[d].x, o);
      acc[d].y += __shfl_xor_sync(0xffffffffu, acc[d].y, o);
    }
}

// x is read with stride xs (xs = batch: one mode's column of the mode-interleaved P).
template <int DIM, class Emit>
__device__ __forceinline__ void saddle_block(const SsOperatorDev& op, int blk, double omega,
                                             const double2* __restrict__ x, Emit&& emit, int xs = 1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nvb = saddle_nvb(op);
  if (blk < nvb) {
    const int grp = lane >> 3, gl = lane & 7;
#pragma unroll 1
    for (int it = 0; it < SPMV_VROWS / 32; ++it) {
      const int r = blk * SPMV_VROWS + it * 32 + warp * 4 + grp;
      const bool ok = r < op.nfree;
      double2 acc[DIM];
      saddle_vel_row_g8<DIM>(op, ok ? r : -1, omega, x, gl, acc, xs);
      if (ok && gl < DIM) {
        double2 v = acc[0];
#pragma unroll
        for (int d = 1; d < DIM; ++d) if (gl == d) v = acc[d];
        emit(r * DIM + gl, v);
      }
    }
  } else {
    const int pb = blk - nvb;
#pragma unroll 1
    for (int it = 0; it < SPMV_PROWS / 8; ++it) {
      const int j = pb * SPMV_PROWS + it * 8 + warp;
      if (j < op.npf) {
        const double2 v = saddle_pres_row<DIM>(op, j, x, lane, xs);
        if (lane == 0) emit(op.nfv + j, v);
      }
    }
  }
}

template <class Emit>
__device__ __forceinline__ void csr_block(const SsCsrDev& A, int set, int blk, const double2* __restrict__ x,
                                          Emit&& emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int it = 0; it < SPMV_PROWS / 8; ++it) {
    const int row = blk * SPMV_PROWS + it * 8 + warp;
    if (row < A.n) {
      const double2 v = csr_row(A, set, row, x, lane);
      if (lane == 0) emit(row, v);
    }
  }
}

__device__ __forceinline__ double2 ldnc2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Mode-interleaved batched SpMV over one row block (the GMRES tick's inner SpMV and the
// standalone ss_spmv_batched_interleaved).  x is [row][ps] (column m = mode m), y is [m][ld].
// Threads walk the block's (row, mode) pairs, mode fastest: matrix loads are broadcasts and the
// x gathers contiguous runs over the batch.  Each (row, mode) is summed by one thread in entry
// order (deterministic, independent of the batch).  active(m) selects modes; scale(m) multiplies.
template <int DIM, class Active, class Omega, class Scale>
__device__ __forceinline__ void saddle_block_interleaved(const SsOperatorDev& op, int blk, int sub, int split,
                                                         int nb, int ps, const double2* __restrict__ x,
                                                         double2* __restrict__ y, int64_t ld, int jacobi,
                                                         Active active, Omega omega_of, Scale scale_of) {
  const int i0 = __ldg(op.sbptr + blk), i1 = __ldg(op.sbptr + blk + 1);
  const int npairs = (i1 - i0) * nb;
  for (int pr = sub * blockDim.x + threadIdx.x; pr < npairs; pr += split * blockDim.x) {
    const int item = __ldg(op.sitems + i0 + pr / nb), m = pr % nb;
    const bool vel = item < op.nfree;
    const int r = vel ? item : item - op.nfree;
    if (!active(m)) continue;
    const double om = omega_of(m), xs = scale_of(m);
    const double2* P = x + m;
    double2* w = y + (size_t)m * ld;
    if (vel) {
      double2 acc[DIM];
#pragma unroll
      for (int d = 0; d < DIM; ++d) acc[d] = make_double2(0.0, 0.0);
      const int e0 = __ldg(op.nptr + r), e1 = __ldg(op.nptr + r + 1);
      int e = e0;
      for (; e + 4 <= e1; e += 4) {
        int B[4];
        double2 sm[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { B[u] = __ldg(op.ncol + e + u); sm[u] = __ldg(op.sm + e + u); }
        double2 v[4][DIM];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int d = 0; d < DIM; ++d) v[u][d] = ldnc2(P + ((size_t)B[u] * DIM + d) * ps);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double am = om * sm[u].y;
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            acc[d].x += sm[u].x * v[u][d].x - am * v[u][d].y;
            acc[d].y += sm[u].x * v[u][d].y + am * v[u][d].x;
          }
        }
      }
      for (; e < e1; ++e) {
        const int B = __ldg(op.ncol + e);
        const double2 sm = __ldg(op.sm + e);
        const double am = om * sm.y;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const double2 v = ldnc2(P + ((size_t)B * DIM + d) * ps);
          acc[d].x += sm.x * v.x - am * v.y;
          acc[d].y += sm.x * v.y + am * v.x;
        }
      }
      const int p0 = __ldg(op.pptr + r), p1 = __ldg(op.pptr + r + 1);
#pragma unroll 4
      for (int q = p0; q < p1; ++q) {
        const double2 v = ldnc2(P + (size_t)(op.nfv + __ldg(op.pcol + q)) * ps);
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const double dv = __ldg(op.dp + (size_t)q * DIM + d);
          acc[d].x += dv * v.x;
          acc[d].y += dv * v.y;
        }
      }
      const double2 sj = jacobi ? saddle_jacobi(op, r, om) : make_double2(1.0, 0.0);
#pragma unroll
      for (int d = 0; d < DIM; ++d) w[(size_t)r * DIM + d] = cmul(sj, cscale(acc[d], xs));
    } else {
      double2 acc = make_double2(0.0, 0.0);
      const int e0 = __ldg(op.tptr + r), e1 = __ldg(op.tptr + r + 1);
#pragma unroll 4
      for (int e = e0; e < e1; ++e) {
        const double2* xb = P + (size_t)__ldg(op.tcol + e) * DIM * ps;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const double dv = __ldg(op.dt + (size_t)e * DIM + d);
          const double2 v = ldnc2(xb + (size_t)d * ps);
          acc.x += dv * v.x;
          acc.y += dv * v.y;
        }
      }
      w[op.nfv + r] = cscale(acc, xs);
    }
  }
}
