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

// Accumulations with pinned rounding.  The CUDA sources are compiled with -fmad=false, so no
// expression is contracted implicitly (the result of a sum never depends on the kernel it is
// inlined into -- the fused tick and the four-kernel tick round identically); the hot loops use
// these explicit FMAs instead.
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  return make_double2(__fma_rn(a.x, b.x, __fma_rn(-a.y, b.y, acc.x)), __fma_rn(a.x, b.y, __fma_rn(a.y, b.x, acc.y)));
}
// acc + conj(a)*b
__device__ __forceinline__ double2 cfmaconj(double2 a, double2 b, double2 acc) {
  return make_double2(__fma_rn(a.x, b.x, __fma_rn(a.y, b.y, acc.x)), __fma_rn(a.x, b.y, __fma_rn(-a.y, b.x, acc.y)));
}
// acc + r*b (real r)
__device__ __forceinline__ double2 rfma(double r, double2 b, double2 acc) {
  return make_double2(__fma_rn(r, b.x, acc.x), __fma_rn(r, b.y, acc.y));
}

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

// ---- TMA bulk copies (cp.async.bulk, global -> shared, completion on an mbarrier) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint64_t* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x-vector loads.  NC = true: the launch never writes x, plain loads (the compiler may take the
// read-only path).  NC = false: the persistent fused tick kernel writes x (P, X) in a later phase of
// the same launch, so x is read with an explicit weak ld.global -- never the non-coherent path,
// whose cache lives for the whole launch; the grid barrier's fences order it.
template <bool NC>
__device__ __forceinline__ double2 ldx(const double2* p) {
  if (NC) return *p;
  double2 v;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Matrix-stream loads of the row-layout SpMV.  SS_MATRIX_LOAD_NA=1 streams the (read-once) matrix
// with ld.global.nc.L1::no_allocate so L1 keeps the x-gather lines; 0 = plain __ldg.
#ifndef SS_MATRIX_LOAD_NA
#define SS_MATRIX_LOAD_NA 0
#endif
__device__ __forceinline__ int ldm(const int* p) {
#if SS_MATRIX_LOAD_NA
  int v;
  asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double ldm(const double* p) {
#if SS_MATRIX_LOAD_NA
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double2 ldm(const double2* p) {
#if SS_MATRIX_LOAD_NA
  double2 v;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

#ifndef SS_PRES_UNROLL
#define SS_PRES_UNROLL 1
#endif
constexpr int PRES_UNROLL = SS_PRES_UNROLL;   // entries per lane of a pressure row loaded per round

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
      acc[d] = cfma(make_double2(a.x, am), v, acc[d]);
    }
  }
  const int p0 = __ldg(op.pptr + r), p1 = __ldg(op.pptr + r + 1);
  for (int e = p0 + lane; e < p1; e += 32) {
    const double2 v = x[op.nfv + __ldg(op.pcol + e)];
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const double dv = __ldg(op.dp + (size_t)e * DIM + d);
      acc[d] = rfma(dv, v, acc[d]);
    }
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    acc[d].x = warp_sum(acc[d].x);
    acc[d].y = warp_sum(acc[d].y);
  }
}

// Pressure row j: sum over free nodes B, components d of D[(B,d),P] x_(B,d).
// Lanes per pressure row of the row-layout SpMV (32: a warp per row; 8 or 16: 4 or 2 rows per warp;
// the 32-row pressure blocks need >= 8).  Config 5 in-cycle: 32 lanes 3.83 ms, 16 3.82, 8 3.66.
#ifndef SS_PRES_LANES
#define SS_PRES_LANES 8
#endif
constexpr int PRES_LANES = SS_PRES_LANES;

// PL lanes (an aligned group) compute pressure row j (j < 0: contributes nothing; every lane of
// the warp must call, the group reduction is an xor butterfly over PL lanes).
template <int DIM, bool NC = true, int PL = 32>
__device__ __forceinline__ double2 saddle_pres_row(const SsOperatorDev& op, int j,
                                                   const double2* __restrict__ x, int lane, int xs = 1) {
  double2 acc = make_double2(0.0, 0.0);
  int e0 = 0, e1 = 0;
  if (j >= 0) { e0 = __ldg(op.tptr + j); e1 = __ldg(op.tptr + j + 1); }
  const int gl = lane % PL;
#pragma unroll PRES_UNROLL
  for (int e = e0 + gl; e < e1; e += PL) {
    const double2* xb = x + (size_t)ldm(op.tcol + e) * DIM * xs;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      const double dv = ldm(op.dt + (size_t)e * DIM + d);
      const double2 v = ldx<NC>(xb + (size_t)d * xs);
      acc = rfma(dv, v, acc);
    }
  }
#pragma unroll
  for (int o = PL / 2; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  return acc;
}

// Generic complex CSR row (drop-in gmres on arbitrary matrices): warp per row.
template <bool NC = true>
__device__ __forceinline__ double2 csr_row(const SsCsrDev& A, int set, int row,
                                           const double2* __restrict__ x, int lane) {
  double2 acc = make_double2(0.0, 0.0);
  const double2* vals = A.vals + (size_t)set * A.nnz;
  const int e0 = __ldg(A.indptr + row), e1 = __ldg(A.indptr + row + 1);
  for (int e = e0 + lane; e < e1; e += 32) {
    const double2 a = __ldg(vals + e);
    const double2 v = ldx<NC>(x + __ldg(A.indices + e));
    acc = cfma(a, v, acc);
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

// Lanes per node row of the row-layout SpMV (4: eight rows per warp).  Config 5 in-cycle (unroll):
// 8 lanes (8) 4.33 ms, 4 lanes (4) 3.80, (2) 4.04, (6) 4.26, 2 lanes (4 / 8) 4.45 / 4.59 (80 registers).
#ifndef SS_ROW_LANES
#define SS_ROW_LANES 4
#endif
constexpr int ROW_LANES = SS_ROW_LANES;
#ifndef SS_ROW_UNROLL
#define SS_ROW_UNROLL 4
#endif
constexpr int ROW_UNROLL = SS_ROW_UNROLL;   // node entries of a lane's row loaded per loop round

// Entry ranges of node row r: {nptr[r], nptr[r+1], pptr[r], pptr[r+1]} (empty for r < 0).
__device__ __forceinline__ int4 row_ranges(const SsOperatorDev& op, int r) {
  if (r < 0) return make_int4(0, 0, 0, 0);
  return make_int4(__ldg(op.nptr + r), __ldg(op.nptr + r + 1), __ldg(op.pptr + r), __ldg(op.pptr + r + 1));
}

template <int DIM, bool NC = true>
__device__ __forceinline__ void saddle_vel_row_g8(const SsOperatorDev& op, int r, double omega,
                                                  const double2* __restrict__ x, int gl, double2 (&acc)[DIM],
                                                  int xs = 1) {
#pragma unroll
  for (int d = 0; d < DIM; ++d) acc[d] = make_double2(0.0, 0.0);
  if (r >= 0) {
    const int4 rg = row_ranges(op, r);   // node and pressure ranges in one load round
    const int e0 = rg.x, e1 = rg.y;
#pragma unroll ROW_UNROLL
    for (int e = e0 + gl; e < e1; e += ROW_LANES) {
      const int B = ldm(op.ncol + e);
      const double2 a = ldm(op.sm + e);
      const double am = omega * a.y;
      const double2* xb = x + (size_t)B * DIM * xs;
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double2 v = ldx<NC>(xb + (size_t)d * xs);
        acc[d] = cfma(make_double2(a.x, am), v, acc[d]);
      }
    }
    const int p0 = rg.z, p1 = rg.w;
#pragma unroll 2
    for (int e = p0 + gl; e < p1; e += ROW_LANES) {
      const double2 v = ldx<NC>(x + (size_t)(op.nfv + ldm(op.pcol + e)) * xs);
#pragma unroll
      for (int d = 0; d < DIM; ++d) {
        const double dv = ldm(op.dp + (size_t)e * DIM + d);
        acc[d] = rfma(dv, v, acc[d]);
      }
    }
  }
#pragma unroll
  for (int o = ROW_LANES / 2; o > 0; o >>= 1)
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      acc[d].x += __shfl_xor_sync(0xffffffffu, acc[d].x, o);
      acc[d].y += __shfl_xor_sync(0xffffffffu, acc[d].y, o);
    }
}

// x is read with stride xs (xs = batch: one mode's column of the mode-interleaved P).
template <int DIM, bool NC = true, class Emit>
__device__ __forceinline__ void saddle_block(const SsOperatorDev& op, int blk, double omega,
                                             const double2* __restrict__ x, Emit&& emit, int xs = 1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nvb = saddle_nvb(op);
  if (blk < nvb) {
    constexpr int RPW = 32 / ROW_LANES;   // rows per warp per iteration
    const int grp = lane / ROW_LANES, gl = lane % ROW_LANES;
    constexpr int ITERS = SPMV_VROWS / (8 * RPW);
    const int rbase = blk * SPMV_VROWS + warp * RPW + grp;
#pragma unroll 1
    for (int it = 0; it < ITERS; ++it) {
      const int r = rbase + it * 8 * RPW;
      const bool ok = r < op.nfree;
      double2 acc[DIM];
      saddle_vel_row_g8<DIM, NC>(op, ok ? r : -1, omega, x, gl, acc, xs);
      if constexpr (ROW_LANES >= DIM) {
        if (ok && gl < DIM) {
          double2 v = acc[0];
#pragma unroll
          for (int d = 1; d < DIM; ++d) if (gl == d) v = acc[d];
          emit(r * DIM + gl, v);
        }
      } else if (ok) {   // fewer lanes than components: lane gl emits components gl, gl + ROW_LANES, ...
#pragma unroll
        for (int d = 0; d < DIM; ++d)
          if (d % ROW_LANES == gl) emit(r * DIM + d, acc[d]);
      }
    }
  } else {
    const int pb = blk - nvb;
    constexpr int PRPW = 32 / PRES_LANES;   // pressure rows per warp per iteration
    static_assert(SPMV_PROWS % (8 * PRPW) == 0 && SPMV_PROWS >= 8 * PRPW, "pressure block must cover whole warps");
#pragma unroll 1
    for (int it = 0; it < SPMV_PROWS / (8 * PRPW); ++it) {
      const int j = pb * SPMV_PROWS + (it * 8 + warp) * PRPW + lane / PRES_LANES;
      const bool ok = j < op.npf;
      const double2 v = saddle_pres_row<DIM, NC, PRES_LANES>(op, ok ? j : -1, x, lane, xs);
      if (ok && lane % PRES_LANES == 0) emit(op.nfv + j, v);
    }
  }
}

template <bool NC = true, class Emit>
__device__ __forceinline__ void csr_block(const SsCsrDev& A, int set, int blk, const double2* __restrict__ x,
                                          Emit&& emit) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int it = 0; it < SPMV_PROWS / 8; ++it) {
    const int row = blk * SPMV_PROWS + it * 8 + warp;
    if (row < A.n) {
      const double2 v = csr_row<NC>(A, set, row, x, lane);
      if (lane == 0) emit(row, v);
    }
  }
}

__device__ __forceinline__ double2 ldnc2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// P gathers of the mode-interleaved SpMV: non-coherent path unless the launch also writes P.
template <bool NC>
__device__ __forceinline__ double2 ldp2(const double2* p) { return NC ? ldnc2(p) : ldx<false>(p); }

#ifndef SS_IL_UNROLL
#define SS_IL_UNROLL 4
#endif
constexpr int IL_U = SS_IL_UNROLL;   // node entries per load round of a (row, mode) thread

// Mode-interleaved batched SpMV over one row block (the GMRES tick's inner SpMV and the
// standalone ss_spmv_batched_interleaved).  x is [row][ps] (column m = mode m), y is [m][ld].
// Threads walk the block's (row, mode) pairs, mode fastest: matrix loads are broadcasts and the
// x gathers contiguous runs over the batch.  Each (row, mode) is summed by one thread in entry
// order (deterministic, independent of the batch).  active(m) selects modes; scale(m) multiplies.
template <int DIM, bool NC = true, class Active, class Omega, class Scale>
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
      for (; e + IL_U <= e1; e += IL_U) {
        int B[IL_U];
        double2 sm[IL_U];
#pragma unroll
        for (int u = 0; u < IL_U; ++u) { B[u] = __ldg(op.ncol + e + u); sm[u] = __ldg(op.sm + e + u); }
        double2 v[IL_U][DIM];
#pragma unroll
        for (int u = 0; u < IL_U; ++u)
#pragma unroll
          for (int d = 0; d < DIM; ++d) v[u][d] = ldp2<NC>(P + ((size_t)B[u] * DIM + d) * ps);
#pragma unroll
        for (int u = 0; u < IL_U; ++u) {
          const double am = om * sm[u].y;
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            acc[d] = cfma(make_double2(sm[u].x, am), v[u][d], acc[d]);
          }
        }
      }
      for (; e < e1; ++e) {
        const int B = __ldg(op.ncol + e);
        const double2 sm = __ldg(op.sm + e);
        const double am = om * sm.y;
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const double2 v = ldp2<NC>(P + ((size_t)B * DIM + d) * ps);
          acc[d] = cfma(make_double2(sm.x, am), v, acc[d]);
        }
      }
      const int p0 = __ldg(op.pptr + r), p1 = __ldg(op.pptr + r + 1);
#pragma unroll 4
      for (int q = p0; q < p1; ++q) {
        const double2 v = ldp2<NC>(P + (size_t)(op.nfv + __ldg(op.pcol + q)) * ps);
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          const double dv = __ldg(op.dp + (size_t)q * DIM + d);
          acc[d] = rfma(dv, v, acc[d]);
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
          const double2 v = ldp2<NC>(xb + (size_t)d * ps);
          acc = rfma(dv, v, acc);
        }
      }
      w[op.nfv + r] = cscale(acc, xs);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// TMA-staged row-layout SpMV (persistent CTAs).  The matrix stream of a chunk of rows -- the
// contiguous ncol/sm/pcol/dp ranges of up to 32 node rows, or tcol/dt of up to 32 pressure rows --
// is moved into a shared-memory stage by bulk copies (cp.async.bulk + mbarrier, a ring of
// STREAM_STAGES stages filled STREAM_STAGES-1 chunks ahead), so the only global loads left in the
// compute loop are the x gathers; the staged chunk is then applied to every active mode.  The
// per-row arithmetic is that of saddle_vel_row_g8 / saddle_pres_row with 8 lanes per node row and
// a warp per pressure row (results equal the row-layout saddle_block's when it is built with
// SS_ROW_LANES=8, SS_PRES_LANES=32; the default row layout now uses 4 / 8 lanes, so the two agree
// to rounding).  Off by default (measured slower).  Chunks (built on the host,
// pattern.cpp) never exceed one stage.
// ------------------------------------------------------------------------------------------------
constexpr int STREAM_STAGE_BYTES = 32768;
constexpr int STREAM_STAGES = 3;
constexpr int STREAM_SMEM = STREAM_STAGES * STREAM_STAGE_BYTES;
constexpr int STREAM_VROWS = 32;   // node rows per velocity chunk (one 8-lane group each)
constexpr int STREAM_PROWS = 32;   // pressure rows per chunk (one warp each, 4 per warp)

struct StreamLayout {
  int e_base, p_base, d_base;            // first staged ncol|tcol index, pcol index, dp|dt double
  int b_col, b_sm, b_pcol, b_d;          // staged bytes of each range (multiples of 16)
  int off_sm, off_pcol, off_d, bytes;    // stage offsets (ncol|tcol at 0)
};

__host__ __device__ __forceinline__ int ss_a16(int v) { return (v + 15) & ~15; }

// ent = {e0, e1, p0, p1}: nptr/pptr ranges of a velocity chunk, or {t0, t1, -, -} (tptr) of a
// pressure chunk.  Start indices are rounded down to 16-byte boundaries (arrays are padded at the end).
__host__ __device__ __forceinline__ StreamLayout stream_layout(int4 ent, bool vel, int dim) {
  StreamLayout L;
  L.e_base = ent.x & ~3;
  L.b_col = ss_a16((ent.y - L.e_base) * 4);
  if (vel) {
    L.b_sm = (ent.y - ent.x) * 16;
    L.p_base = ent.z & ~3;
    L.b_pcol = ss_a16((ent.w - L.p_base) * 4);
    L.d_base = (ent.z * dim) & ~1;
    L.b_d = ss_a16((ent.w * dim - L.d_base) * 8);
  } else {
    L.b_sm = 0;
    L.p_base = 0;
    L.b_pcol = 0;
    L.d_base = (ent.x * dim) & ~1;
    L.b_d = ss_a16((ent.y * dim - L.d_base) * 8);
  }
  L.off_sm = L.b_col;
  L.off_pcol = L.off_sm + L.b_sm;
  L.off_d = L.off_pcol + L.b_pcol;
  L.bytes = L.off_d + L.b_d;
  return L;
}

// Persistent streaming pass over all chunks for every mode m < nb with active(m):
//   x_of(m) -> const double2* (x of mode m, element stride xs), omega_of(m), emit(m, row, value).
template <int DIM, class Active, class Omega, class XOf, class Emit>
__device__ __forceinline__ void saddle_stream(const SsOperatorDev& op, int nb, int xs, unsigned char* ring,
                                              uint64_t* bar, Active active, Omega omega_of, XOf x_of, Emit emit) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x, ncta = gridDim.x;
  const int nmine = cta < op.nchunk ? (op.nchunk - cta + ncta - 1) / ncta : 0;
  if (tid < STREAM_STAGES) mbar_init(&bar[tid], 1);
  fence_mbar_init();
  __syncthreads();
  auto load = [&](int ci) {   // single producer thread
    const int c = cta + ci * ncta;
    const bool vel = c < op.nvchunk;
    const int4 ent = op.cent[c];
    const StreamLayout L = stream_layout(ent, vel, DIM);
    unsigned char* st = ring + (size_t)(ci % STREAM_STAGES) * STREAM_STAGE_BYTES;
    uint64_t* b = &bar[ci % STREAM_STAGES];
    mbar_expect_tx(b, (unsigned)L.bytes);
    if (vel) {
      if (L.b_col) bulk_g2s(st, op.ncol + L.e_base, (unsigned)L.b_col, b);
      if (L.b_sm) bulk_g2s(st + L.off_sm, op.sm + ent.x, (unsigned)L.b_sm, b);
      if (L.b_pcol) bulk_g2s(st + L.off_pcol, op.pcol + L.p_base, (unsigned)L.b_pcol, b);
      if (L.b_d) bulk_g2s(st + L.off_d, op.dp + L.d_base, (unsigned)L.b_d, b);
    } else {
      if (L.b_col) bulk_g2s(st, op.tcol + L.e_base, (unsigned)L.b_col, b);
      if (L.b_d) bulk_g2s(st + L.off_d, op.dt + L.d_base, (unsigned)L.b_d, b);
    }
  };
  if (tid == 0)
    for (int ci = 0; ci < STREAM_STAGES - 1 && ci < nmine; ++ci) load(ci);
  for (int ci = 0; ci < nmine; ++ci) {
    if (tid == 0 && ci + STREAM_STAGES - 1 < nmine) load(ci + STREAM_STAGES - 1);   // stage of chunk ci-1
    const int c = cta + ci * ncta;
    const bool vel = c < op.nvchunk;
    const int4 ent = __ldg(op.cent + c);
    const int2 rows = __ldg(op.crow + c);
    const StreamLayout L = stream_layout(ent, vel, DIM);
    const unsigned char* st = ring + (size_t)(ci % STREAM_STAGES) * STREAM_STAGE_BYTES;
    if (vel) {
      const int grp = tid >> 3, gl = tid & 7;
      const int r = rows.x + grp;
      const bool ok = r < rows.y;
      int e0 = 0, e1 = 0, q0 = 0, q1 = 0;
      if (ok) {   // row ranges: global loads issued before the stage wait
        e0 = __ldg(op.nptr + r); e1 = __ldg(op.nptr + r + 1);
        q0 = __ldg(op.pptr + r); q1 = __ldg(op.pptr + r + 1);
      }
      mbar_wait(&bar[ci % STREAM_STAGES], (unsigned)((ci / STREAM_STAGES) & 1));
      const int* scol = reinterpret_cast<const int*>(st) - L.e_base;
      const double2* ssm = reinterpret_cast<const double2*>(st + L.off_sm) - ent.x;
      const int* spcol = reinterpret_cast<const int*>(st + L.off_pcol) - L.p_base;
      const double* sdp = reinterpret_cast<const double*>(st + L.off_d) - L.d_base;
      for (int m = 0; m < nb; ++m) {
        if (!active(m)) continue;
        const double omega = omega_of(m);
        const double2* __restrict__ x = x_of(m);
        double2 acc[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) acc[d] = make_double2(0.0, 0.0);
#pragma unroll 4
        for (int e = e0 + gl; e < e1; e += 8) {
          const int B = scol[e];
          const double2 a = ssm[e];
          const double am = omega * a.y;
          const double2* xb = x + (size_t)B * DIM * xs;
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            const double2 v = xb[(size_t)d * xs];
            acc[d] = cfma(make_double2(a.x, am), v, acc[d]);
          }
        }
#pragma unroll 2
        for (int e = q0 + gl; e < q1; e += 8) {
          const double2 v = x[(size_t)(op.nfv + spcol[e]) * xs];
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            const double dv = sdp[(size_t)e * DIM + d];
            acc[d] = rfma(dv, v, acc[d]);
          }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1)
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            acc[d].x += __shfl_xor_sync(0xffffffffu, acc[d].x, o);
            acc[d].y += __shfl_xor_sync(0xffffffffu, acc[d].y, o);
          }
        if (ok && gl < DIM) {
          double2 v = acc[0];
#pragma unroll
          for (int d = 1; d < DIM; ++d) if (gl == d) v = acc[d];
          emit(m, r * DIM + gl, v);
        }
      }
    } else {
      int t0[STREAM_PROWS / 8], t1[STREAM_PROWS / 8];
#pragma unroll
      for (int it = 0; it < STREAM_PROWS / 8; ++it) {
        const int j = rows.x + it * 8 + warp;
        t0[it] = j < rows.y ? __ldg(op.tptr + j) : 0;
        t1[it] = j < rows.y ? __ldg(op.tptr + j + 1) : 0;
      }
      mbar_wait(&bar[ci % STREAM_STAGES], (unsigned)((ci / STREAM_STAGES) & 1));
      const int* scol = reinterpret_cast<const int*>(st) - L.e_base;
      const double* sdt = reinterpret_cast<const double*>(st + L.off_d) - L.d_base;
      for (int m = 0; m < nb; ++m) {
        if (!active(m)) continue;
        const double2* __restrict__ x = x_of(m);
#pragma unroll 1
        for (int it = 0; it < STREAM_PROWS / 8; ++it) {
          const int j = rows.x + it * 8 + warp;
          if (j >= rows.y) break;
          double2 acc = make_double2(0.0, 0.0);
          for (int e = t0[it] + lane; e < t1[it]; e += 32) {
            const double2* xb = x + (size_t)scol[e] * DIM * xs;
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
              const double dv = sdt[(size_t)e * DIM + d];
              const double2 v = xb[(size_t)d * xs];
              acc = rfma(dv, v, acc);
            }
          }
          acc.x = warp_sum(acc.x);
          acc.y = warp_sum(acc.y);
          if (lane == 0) emit(m, op.nfv + j, acc);
        }
      }
    }
    fence_proxy_async();   // generic-proxy reads of this stage before the async proxy refills it
    __syncthreads();
  }
}
