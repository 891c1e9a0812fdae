// Mode-batched, device-resident restarted GMRES(m) with left Jacobi preconditioning and CGS2.
//
// Restates the reference solver gmres (pkg/src/spectralstokes/krylov.py:63-164) for a batch of
// independent modes.  Semantics kept exactly (SURVEY.md §8a'): same restart, classical Gram-
// Schmidt with one reorthogonalisation (H column = c + c2), complex Givens rotations, the
// est <= tol*||s.b|| inner exit, the true-residual re-check at every cycle end, the x0.25 target
// tightening, happy/denominator breakdowns and maxiter counted in inner iterations.  Allowed
// re-associations only: w -= Qc fused with c2 = Q^H w (3 basis passes instead of 4), deferred
// 1/||w|| scaling of stored basis vectors, mode-major storage.
//
// Execution model: each mode carries a small device state machine (ModeCtl.phase).  One "tick"
// is a fixed sequence of four kernels over the whole batch, captured in a CUDA graph:
//   spmv   INNER/START: w = s.(A q_k)          RESID: t = b - A x, r = s.t, norms, cycle decisions
//   passA  INNER: c  = Q^H w                    (partials per segment, last CTA reduces)
//          XUPDATE: x += Q y                    (cycle end; own k_pass<PASS_X> launch if SS_X_IN_A=0)
//   passB  INNER: w -= Q c ; c2 = Q^H w         (one read of Q for both)
//   passC  INNER: w -= Q c2 ; Q[k+1] = P = w ; ||w|| -> last CTA: Givens, estimate, exit tests,
//                 triangular solve at cycle end
// Every state change is made by the last CTA of a mode in a kernel (the tick SpMV: the last CTA
// of the grid, for all modes), so all CTAs of a mode see a consistent phase.  The reduction structure of a mode depends only on (n, k, restart), never on
// which other modes share the batch: per-mode results are bitwise invariant under batching and
// mode order (the reference's test_spectral.py:187-205 contract).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <string>
#include <vector>

#include "ss_common.h"
#include "ss_pattern.h"
#include "ss_spmv.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

enum Phase : int { PH_IDLE = 0, PH_RESID = 1, PH_START = 2, PH_INNER = 3, PH_XUPDATE = 4, PH_DONE = 5 };

struct ModeCtl {
  int phase, k, iters, maxiter;
  int restart, breakdown, first, converged;
  int zero_x, set, hist_len, done_tick;   // done_tick: tick at which the mode finished
  double beta, target, bnorm, tol;
  double omega, true_res, gk_last, est;
};

constexpr int PT = 256;        // threads per CTA for every Krylov kernel
constexpr int PASS_MAX_STAGES = 8;
constexpr int PASS_L2_AHEAD = 4;          // chunks prefetched into L2 beyond the smem ring
constexpr int PASS_SMEM_ELEMS = 13440;    // dynamic shared memory of a basis pass (210 KB)
constexpr int WIDE_RESTART = 240;         // largest restart served by the TMA-ring passes (J <= 241)

struct KArgs {
  int kind;                    // 0 saddle, 1 csr
  int nb, n, restart, jcap;
  int64_t ld;
  int nseg, seg_rows;          // pass segmentation (depends on n only)
  int nsb;                     // spmv blocks per mode
  int smem_elems;              // double2 capacity of the basis-pass pipeline ring
  int stage_div;               // a stage may use smem_elems / stage_div
  int jacobi;
  int64_t hist_cap;
  SsOperatorDev op;
  SsCsrDev csr;
  ModeCtl* ctl;
  double2 *Q, *W, *X, *RHS;
  double2* P;                  // current raw basis vectors, mode-interleaved [row][pstride] (SpMV input)
  int pstride;                 // = max batch
  int spmv_split;              // sub-CTAs per SpMV row block (fills the GPU when n is small)
  int nblk;                    // ld / RB row blocks; Q is row-block-major: [b][blk][jcap][RB]
  double* qs;                  // [b][jcap] scale of raw basis vectors
  double2 *H, *G, *CS, *SN, *C1, *C2, *Y;
  double2* part;               // [b][nseg][jcap] pass partials
  double2* spart;              // [b][nsb] spmv partials (x: ||t||^2, y: ||r||^2)
  int* counters;               // [b][8]
  int* n_done;
  double* hist;                // [b][hist_cap]
  unsigned long long* bytes;   // [8] algorithmic bytes moved per kernel kind (profiling)
  long long* loop;             // [0] ticks executed by the device-side loop, [1] tick cap, [2] ticks of this solve
  int x_in_a;                  // cycle-end x update inside the next tick's pass-A launch (1) or own launch (0)
  int gthr[3];                 // pass B: largest J using 1, 2, 4 warps per row block (8 above)
  int row_spmv;                // tick SpMV: per-mode 8-lanes-per-row blocks (n >= SS_ROW_SPMV_N) instead of interleaved
  int wide;                    // restart > WIDE_RESTART: basis passes without the shared-memory ring (any J)
  int stream_spmv;             // row layout: TMA-staged persistent SpMV (1) or one CTA per row block (0)
  int fused;                   // running inside k_tick_fused (persistent, grid barriers between phases)
  int row_dyn;                 // row-layout tick SpMV: blocks dealt from an atomic counter (SS_ROW_DYN)
  int ahead_bytes;             // basis-pass prefetch cap (bytes in flight per CTA; 0 = the whole ring)
  int pass_alt;                // basis passes stream their segment in alternating directions (SS_PASS_ALT)
  long long* ptime;            // fused-kernel phase timestamps [tick % FUSED_PROF_TICKS][5] (SS_FUSED_PROF)
};
constexpr int FUSED_PROF_TICKS = 1 << 16;

constexpr int RB = 32;         // rows per block of the row-block-major basis layout

// Basis storage is row-block-major: for every block of RB rows the J basis vectors are
// contiguous (J x 512 B), so a basis pass streams long contiguous runs from HBM and moves a
// whole block with ONE bulk-TMA copy.
__device__ __forceinline__ double2* qblock(const KArgs& a, int b, int blk) {
  return a.Q + ((size_t)b * a.nblk + blk) * a.jcap * RB;
}
__device__ __forceinline__ double2& qat(const KArgs& a, int b, int j, int64_t row) {
  return qblock(a, b, (int)(row / RB))[(size_t)j * RB + (row % RB)];
}

// Last-CTA election: returns true in every thread of the CTA that finished last for this mode.
__device__ __forceinline__ bool last_cta(const KArgs& a, int b, int which, int total, int* sflag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int t = atomicAdd(a.counters + b * 8 + which, 1);
    *sflag = (t == total - 1);
    if (*sflag) a.counters[b * 8 + which] = 0;
  }
  __syncthreads();
  const bool last = *sflag;
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ void mark_done(const KArgs& a, ModeCtl* c, int converged) {
  c->phase = PH_DONE;
  c->done_tick = (int)a.loop[2];
  c->converged = converged;
  atomicAdd(a.n_done, 1);
}

// ------------------------------------------------------------------------------------------------
// Row scale s_i (Jacobi) for either operator kind.
// ------------------------------------------------------------------------------------------------
template <int DIM>
__device__ __forceinline__ double2 row_scale(const KArgs& a, int b, int row, double om) {
  if (!a.jacobi) return make_double2(1.0, 0.0);
  if (a.kind == 0) return row < a.op.nfv ? saddle_jacobi(a.op, row / DIM, om) : make_double2(1.0, 0.0);
  return a.csr.scale ? a.csr.scale[(size_t)(a.csr.nvals > 1 ? b : 0) * a.csr.n + row] : make_double2(1.0, 0.0);
}

// ------------------------------------------------------------------------------------------------
// Init: ||b||, target = tol*||s.b||; phase RESID (krylov.py:71-80).
// ------------------------------------------------------------------------------------------------
template <int DIM>
__global__ void __launch_bounds__(PT) k_init(KArgs a) {
  __shared__ double red[2][PT];
  __shared__ int sflag;
  const int b = blockIdx.x / a.nseg, s = blockIdx.x % a.nseg;
  if (b >= a.nb) return;
  ModeCtl* c = a.ctl + b;
  const double om = c->omega;
  const double2* rhs = a.RHS + (size_t)b * a.ld;
  const int r0 = s * a.seg_rows, r1 = min((int64_t)(s + 1) * a.seg_rows, (int64_t)a.n);
  double bb = 0, sb = 0;
  for (int i = r0 + threadIdx.x; i < r1; i += PT) {
    const double2 v = rhs[i];
    bb += cabs2(v);
    sb += cabs2(cmul(row_scale<DIM>(a, b, i, om), v));
  }
  red[0][threadIdx.x] = bb;
  red[1][threadIdx.x] = sb;
  __syncthreads();
  for (int o = PT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red[0][threadIdx.x] += red[0][threadIdx.x + o];
      red[1][threadIdx.x] += red[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  double2* part = a.part + ((size_t)b * a.nseg) * a.jcap;
  if (threadIdx.x == 0) part[(size_t)s * a.jcap] = make_double2(red[0][0], red[1][0]);
  if (!last_cta(a, b, 5, a.nseg, &sflag)) return;
  if (threadIdx.x == 0) {
    double t0 = 0, t1 = 0;
    for (int q = 0; q < a.nseg; ++q) {
      const double2 v = __ldcg(part + (size_t)q * a.jcap);
      t0 += v.x;
      t1 += v.y;
    }
    c->bnorm = sqrt(t0);
    c->k = 0;
    c->iters = 0;
    c->breakdown = 0;
    c->first = 1;
    c->converged = 0;
    c->zero_x = 0;
    c->hist_len = 0;
    c->true_res = 0;
    c->est = 0;
    if (c->bnorm == 0.0) {          // krylov.py:73-75: x = 0, 0 iterations, converged
      c->zero_x = 1;
      mark_done(a, c, 1);
    } else {
      c->target = c->tol * sqrt(t1);
      c->phase = PH_RESID;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Tick kernel 1: SpMV (inner w = s.(A q_k)) or residual (t = b - A x, r = s.t) + cycle decisions.
//
// The current raw basis vectors of all modes live in P with a MODE-INTERLEAVED layout
// P[row * pstride + mode]: one gather of node B's component d returns that value for every mode
// of the batch as one contiguous run, so a warp whose lanes are modes issues coalesced gathers
// and shares every matrix-entry load (broadcast) across the batch.  Each lane owns one
// (row, mode) pair and sums the row's entries sequentially: no cross-lane reduction, and a
// mode's result never depends on the other modes in the batch.
// ------------------------------------------------------------------------------------------------
constexpr int MAXB_SMEM = 256;   // modes whose per-tick state is cached in shared memory

template <int DIM, bool NC>
__device__ __forceinline__ void spmv_inner_interleaved(const KArgs& a, int blk, int sub, const int* sph,
                                                       const double* som, const double* sxs) {
  saddle_block_interleaved<DIM, NC>(
      a.op, blk, sub, a.spmv_split, a.nb, a.pstride, a.P, a.W, a.ld, a.jacobi,
      [&](int m) { return sph[m] == PH_INNER || sph[m] == PH_START; },
      [&](int m) { return som[m]; }, [&](int m) { return sxs[m]; });
}

// RESID for one mode (row layout X): t = b - A x, r = s.t -> P (interleaved) and Q[0]; norms.
template <int DIM, bool NC = true>
__device__ __forceinline__ void spmv_resid_mode(const KArgs& a, int b, int sb, double om) {
  __shared__ double red[2][PT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2* x = a.X + (size_t)b * a.ld;
  const double2* rhs = a.RHS + (size_t)b * a.ld;
  double tt = 0, rr = 0;
  auto emit = [&](int row, double2 v) {
    const double2 s = row_scale<DIM>(a, b, row, om);
    const double2 t = csub(rhs[row], v);
    const double2 r = cmul(s, t);
    a.P[(size_t)row * a.pstride + b] = r;
    qat(a, b, 0, row) = r;
    tt += cabs2(t);
    rr += cabs2(r);
  };
  if (a.kind == 0) saddle_block<DIM, NC>(a.op, sb, om, x, emit);
  else csr_block<NC>(a.csr, a.csr.nvals > 1 ? b : 0, sb, x, emit);
  tt = warp_sum(tt);
  rr = warp_sum(rr);
  if (lane == 0) { red[0][warp] = tt; red[1][warp] = rr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0;
    for (int w = 0; w < PT / 32; ++w) { s0 += red[0][w]; s1 += red[1][w]; }
    a.spart[(size_t)b * a.nsb + sb] = make_double2(s0, s1);
  }
  __syncthreads();
}

// Generic-CSR inner SpMV for one mode (row layout through P column b).
__device__ __forceinline__ void spmv_inner_csr_mode(const KArgs& a, int b, int sb, double xs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SsCsrDev& A = a.csr;
  const int set = A.nvals > 1 ? b : 0;
  const double2* vals = A.vals + (size_t)set * A.nnz;
  for (int it = 0; it < SPMV_PROWS / 8; ++it) {
    const int row = sb * SPMV_PROWS + it * 8 + warp;
    if (row >= A.n) break;
    double2 acc = make_double2(0.0, 0.0);
    for (int e = A.indptr[row] + lane; e < A.indptr[row + 1]; e += 32) {
      const double2 av = vals[e];
      const double2 v = a.P[(size_t)A.indices[e] * a.pstride + b];
      acc = cfma(av, v, acc);
    }
    acc.x = warp_sum(acc.x);
    acc.y = warp_sum(acc.y);
    if (lane == 0) {
      const double2 s = A.scale && a.jacobi ? A.scale[(size_t)set * A.n + row] : make_double2(1.0, 0.0);
      a.W[(size_t)b * a.ld + row] = cmul(s, cscale(acc, xs));
    }
  }
}

// Cycle-boundary decisions of mode b once every CTA has contributed (krylov.py:93-103,155-162).
// Called by the last CTA of the tick SpMV for every mode it touched.
__device__ __forceinline__ void spmv_finalize_mode(const KArgs& a, int b, int phase, double2* rsum) {
  ModeCtl* c = a.ctl + b;
  if (phase != PH_RESID) {
    if (threadIdx.x == 0 && phase == PH_START) c->phase = PH_INNER;
    __syncthreads();
    return;
  }
  double2 acc = make_double2(0.0, 0.0);
  for (int q = threadIdx.x; q < a.nsb; q += PT) {
    const double2 v = __ldcg(a.spart + (size_t)b * a.nsb + q);
    acc.x += v.x;
    acc.y += v.y;
  }
  rsum[threadIdx.x] = acc;
  __syncthreads();
  for (int o = PT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) rsum[threadIdx.x] = cadd(rsum[threadIdx.x], rsum[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tn = sqrt(rsum[0].x), rn = sqrt(rsum[0].y);
    bool done = false;
    if (!c->first) {
      c->true_res = tn / c->bnorm;
      if (c->true_res <= c->tol) { mark_done(a, c, 1); done = true; }
      else if (c->breakdown) { mark_done(a, c, 0); done = true; }
      else if (c->gk_last <= c->target) c->target *= 0.25;
    }
    if (!done) {
      if (c->iters >= c->maxiter) {
        mark_done(a, c, 0);
      } else if (rn == 0.0) {
        mark_done(a, c, 1);
      } else {
        c->beta = rn;
        c->k = 0;
        c->breakdown = 0;
        c->first = 0;
        a.qs[b * a.jcap] = 1.0 / rn;
        c->phase = PH_START;
      }
    }
  }
  __syncthreads();
  if (c->phase == PH_START) {
    double2* g = a.G + (size_t)b * a.jcap;
    for (int j = threadIdx.x; j < a.jcap; j += PT) g[j] = make_double2(j == 0 ? c->beta : 0.0, 0.0);
  }
  __syncthreads();
}

// Staged row-layout tick SpMV: true when the tick runs the persistent TMA-staged kernel.
__host__ __device__ __forceinline__ bool tick_streamed(const KArgs& a) {
  return a.kind == 0 && a.row_spmv && a.stream_spmv && a.op.nchunk > 0;
}

// Streamed row layout (tick_streamed): persistent CTAs walk the TMA-staged chunks for the
// INNER/START modes, then the fixed row blocks grid-stride for RESID modes (per-block partials in
// the same fixed tree as k_tick_spmv), then one last-CTA election makes the cycle decisions.
template <int DIM>
__global__ void __launch_bounds__(PT, 2) k_tick_spmv_stream(KArgs a) {
  __shared__ int sph[MAXB_SMEM];
  __shared__ double som[MAXB_SMEM], sxs[MAXB_SMEM];
  __shared__ int sflag, s_any_inner;
  __shared__ double2 rsum[PT];
  extern __shared__ __align__(128) unsigned char sring[];
  __shared__ __align__(8) uint64_t sbar[STREAM_STAGES];
  if (threadIdx.x == 0) s_any_inner = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < a.nb; b += PT) {
    const ModeCtl* c = a.ctl + b;
    const int ph = c->phase;
    sph[b] = ph;
    som[b] = c->omega;
    sxs[b] = (ph == PH_INNER || ph == PH_START) ? a.qs[b * a.jcap + c->k] : 0.0;
    if (ph == PH_INNER || ph == PH_START) s_any_inner = 1;
  }
  __syncthreads();
  if (s_any_inner)
    saddle_stream<DIM>(
        a.op, a.nb, a.pstride, sring, sbar, [&](int m) { return sph[m] == PH_INNER || sph[m] == PH_START; },
        [&](int m) { return som[m]; }, [&](int m) { return (const double2*)a.P + m; },
        [&](int m, int row, double2 v) {
          const double om = som[m];
          const double2 s = row < a.op.nfv && a.jacobi ? saddle_jacobi(a.op, row / DIM, om) : make_double2(1.0, 0.0);
          a.W[(size_t)m * a.ld + row] = cmul(s, cscale(v, sxs[m]));
        });
  for (int sb = blockIdx.x; sb < a.nsb; sb += gridDim.x)
    for (int b = 0; b < a.nb; ++b)
      if (sph[b] == PH_RESID) spmv_resid_mode<DIM>(a, b, sb, som[b]);
  if (!last_cta(a, 0, 6, (int)gridDim.x, &sflag)) return;
  if (threadIdx.x == 0) a.loop[2] += 1;   // one tick done (per-mode completion ticks, ss_krylov_done_ticks)
  for (int b = 0; b < a.nb; ++b) {
    const int ph = sph[b];
    if (ph == PH_INNER || ph == PH_START || ph == PH_RESID) spmv_finalize_mode(a, b, ph, rsum);
  }
}

// Tick SpMV over virtual block vb of nvb (a kernel launch: blockIdx.x of gridDim.x; the fused
// persistent kernel: its CTAs walk the virtual blocks).  Shared state is passed in so that the
// fused kernel declares it once.
template <int DIM, int ROW, bool NC>
__device__ __forceinline__ void tick_spmv_body(const KArgs& a, int vb, int nvb, int* sph, double* som, double* sxs,
                                               int* sflag, int* s_any_inner, double2* rsum) {
  const int sb = vb / a.spmv_split, sub = vb % a.spmv_split;
  if (a.fused) __syncthreads();   // shared state of the previous virtual block
  if (threadIdx.x == 0) *s_any_inner = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < a.nb; b += PT) {
    const ModeCtl* c = a.ctl + b;
    const int ph = c->phase;
    sph[b] = ph;
    som[b] = c->omega;
    sxs[b] = (ph == PH_INNER || ph == PH_START) ? a.qs[b * a.jcap + c->k] : 0.0;
    if (ph == PH_INNER || ph == PH_START) *s_any_inner = 1;
  }
  __syncthreads();
  if (ROW) {
    // very large n (rule on n only, so per-mode results stay batch-invariant; at most a few modes
    // fit a GPU there): 8 lanes per node row with a warp reduction, one mode at a time, reading
    // the mode's column of P with stride pstride.  Grid-stride over the row blocks (a few CTAs per
    // SM): the mode-state prologue and the last-CTA election are paid per CTA, not per block.
    const int b0 = vb, b1 = a.nsb, bstep = nvb;   // blocks dealt round-robin (row_dyn = 0)
    __shared__ int s_next;
    int blk = b0;
    if (a.row_dyn) {   // option: blocks dealt in order from an atomic counter (compact window)
      if (threadIdx.x == 0) s_next = atomicAdd(a.counters + 7, 1);
      __syncthreads();
      blk = s_next;
    }
    for (; blk < b1;) {
      if (a.row_dyn) {
        __syncthreads();   // every thread has read s_next
        if (threadIdx.x == 0) s_next = atomicAdd(a.counters + 7, 1);   // next index, fetched during this block
      }
      if (*s_any_inner)
        for (int b = 0; b < a.nb; ++b) {
          if (sph[b] != PH_INNER && sph[b] != PH_START) continue;
          const double om = som[b], xs = sxs[b];
          double2* w = a.W + (size_t)b * a.ld;
          saddle_block<DIM, NC>(a.op, blk, om, a.P + b, [&](int row, double2 v) {
            const double2 s = row < a.op.nfv && a.jacobi ? saddle_jacobi(a.op, row / DIM, om) : make_double2(1.0, 0.0);
            w[row] = cmul(s, cscale(v, xs));
          }, a.pstride);
        }
      for (int b = 0; b < a.nb; ++b)
        if (sph[b] == PH_RESID) spmv_resid_mode<DIM, NC>(a, b, blk, som[b]);
      if (a.row_dyn) {
        __syncthreads();
        blk = s_next;
      } else {
        blk += bstep;
      }
    }
  } else if (*s_any_inner) {
    if (a.kind == 0) {
      spmv_inner_interleaved<DIM, NC>(a, sb, sub, sph, som, sxs);
    } else {
      if (sub == 0)
        for (int b = 0; b < a.nb; ++b)
          if (sph[b] == PH_INNER || sph[b] == PH_START) spmv_inner_csr_mode(a, b, sb, sxs[b]);
    }
  }
  if (!ROW && sub == 0)   // residual rows of the block are owned by its first sub-CTA (fixed reduction tree)
    for (int b = 0; b < a.nb; ++b)
      if (sph[b] == PH_RESID) spmv_resid_mode<DIM, NC>(a, b, sb, som[b]);
  // one election for the whole batch (slot 6 of mode 0's counters): the last CTA to finish makes
  // every mode's cycle decisions
  if (!last_cta(a, 0, 6, nvb, sflag)) return;
  if (threadIdx.x == 0) {
    a.loop[2] += 1;
    if (ROW && a.row_dyn) a.counters[7] = 0;   // dynamic block counter, for the next launch
  }   // one tick done (per-mode completion ticks, ss_krylov_done_ticks)
  for (int b = 0; b < a.nb; ++b) {
    const int ph = sph[b];
    if (ph == PH_INNER || ph == PH_START || ph == PH_RESID) spmv_finalize_mode(a, b, ph, rsum);
  }
}

// One CTA = one row block, all modes of the batch.  ROW: the row-layout INNER SpMV (8 lanes per
// node row, the mode's strided column of P), instantiated separately so its register allocation is
// not shaped by the mode-interleaved kernel.
// Launch bounds: maxThreads only (ptxas then keeps these kernels at 64 registers, 4 CTAs per SM;
// an explicit minBlocks of 1 lets it take ~128 and costs 1.5x in-cycle at config 5).
#ifdef SS_TICK_MINB
#define SS_TICK_BOUNDS __launch_bounds__(PT, SS_TICK_MINB)
#else
#define SS_TICK_BOUNDS __launch_bounds__(PT)
#endif
template <int DIM, int ROW>
__global__ void SS_TICK_BOUNDS k_tick_spmv(KArgs a) {
  __shared__ int sph[MAXB_SMEM];
  __shared__ double som[MAXB_SMEM], sxs[MAXB_SMEM];
  __shared__ int sflag, s_any_inner;
  __shared__ double2 rsum[PT];
  tick_spmv_body<DIM, ROW, true>(a, blockIdx.x, gridDim.x, sph, som, sxs, &sflag, &s_any_inner, rsum);
}

// ------------------------------------------------------------------------------------------------
// Basis-streaming passes.  A CTA owns one fixed segment of rows of one mode and streams the
// (J x rows) slab of raw basis vectors through shared memory in chunks (bulk TMA into a ring of
// mbarrier-tracked stages, see stream_segment).
// ------------------------------------------------------------------------------------------------
enum PassKind : int { PASS_A = 1, PASS_B = 2, PASS_C = 3, PASS_X = 4 };

// TMA bulk-copy / mbarrier helpers: ss_spmv.cuh

// Chunks kept in flight ahead of the consumer: the ring's NS - 1, capped at a.ahead_bytes (bulk
// reads stream fastest with ~50-100 KB in flight per SM, tools/probes/read_bw.cu); never below
// one.  Only the issue time of the copies changes, not the chunking: sums are unaffected.
__device__ __forceinline__ int pass_ahead(const KArgs& a, int NS, int stage_elems) {
  int ah = NS - 1;
  if (a.ahead_bytes > 0) ah = min(ah, max(1, a.ahead_bytes / (stage_elems * 16)));
  return max(ah, NS > 1 ? 1 : 0);
}

__device__ __forceinline__ int pass_slices(int nr) { return nr > 4 ? 1 : nr > 2 ? 2 : nr > 1 ? 4 : 8; }

// Streams one segment (SEGB row blocks) of one mode's basis through a ring of shared-memory
// stages filled by bulk TMA (one copy per row block: J x 512 B contiguous, one for the vector).
//   phase 1 (B, C, X): V <- V -/+ sum_j S_j c_j   warps = (block, j-slice), lanes = rows
//   phase 2 (A, B):    acc_t += conj(S_{warp+8t}) V   per-lane register accumulators
// Writes this CTA's partials: part[j] (A, B) or part[0].x = ||w||^2 (C).
template <int PASS, int T>
__device__ __forceinline__ void stream_segment(const KArgs& a, int b, int s, int J, int k, const double2* coef,
                                               double2* smem, uint64_t* mbar, double2* red, double2* part,
                                               bool rev = false) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int segb = a.seg_rows / RB;
  const int blk_begin = s * segb;
  const int blk_end = min(blk_begin + segb, a.nblk);
  const int nblocks = blk_end - blk_begin;
  const int belem = J * RB;
  // passes with an update phase amortise their extra barriers over bigger chunks (measured)
  const int div = a.stage_div > 0 ? a.stage_div : (PASS == PASS_A ? 3 : 2);
  // pass B keeps each thread's basis values in registers between its two phases: one block/chunk
  const int CB = PASS == PASS_B ? 1 : max(1, min(min(nblocks, 8), (a.smem_elems / div) / (belem + RB)));
  const int stage_elems = CB * (belem + RB);
  const int NS = max(1, min(PASS_MAX_STAGES, a.smem_elems / stage_elems));
  const int AH = pass_ahead(a, NS, stage_elems);
  const int nchunks = (nblocks + CB - 1) / CB;
  double2* vec = (PASS == PASS_X ? a.X : a.W) + (size_t)b * a.ld;
  auto stage = [&](int ci) { return smem + (size_t)(ci % NS) * stage_elems; };
  auto load_chunk = [&](int ci) {   // single producer thread
    double2* st = stage(ci);
    const int c0 = blk_begin + (rev ? nchunks - 1 - ci : ci) * CB;
    const int nc = min(CB, blk_end - c0);
    uint64_t* bar = &mbar[ci % NS];
    mbar_expect_tx(bar, (unsigned)(nc * (belem + RB) * 16));
    for (int c = 0; c < nc; ++c) bulk_g2s(st + c * belem, qblock(a, b, c0 + c), (unsigned)belem * 16u, bar);
    bulk_g2s(st + CB * belem, vec + (size_t)c0 * RB, (unsigned)(nc * RB * 16), bar);
  };
  if (tid < PASS_MAX_STAGES) mbar_init(&mbar[tid], 1);
  fence_mbar_init();
  __syncthreads();
  if (tid == 0)
    for (int ci = 0; ci < AH && ci < nchunks; ++ci) load_chunk(ci);
  double2 acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = make_double2(0.0, 0.0);
  double nrm = 0.0;
  for (int ci = 0; ci < nchunks; ++ci) {
    if (tid == 0 && ci + AH < nchunks) load_chunk(ci + AH);   // stage of chunk ci+AH-NS <= ci-1 (released)
    mbar_wait(&mbar[ci % NS], (unsigned)((ci / NS) & 1));
    double2* st = stage(ci);
    const int c0 = blk_begin + (rev ? nchunks - 1 - ci : ci) * CB;
    const int nc = min(CB, blk_end - c0);
    double2* Vb = st + CB * belem;
    if (PASS == PASS_B) {
      // phase 1 with the phase-2 distribution (j = warp + 8t, lane = row): Q read from smem once
      double2 qv[T];
      const double2* S = st + lane;
      double2 p = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = warp + 8 * t;
        if (j < J) {
          qv[t] = S[j * RB];
          const double2 cf = coef[j];
          p = cfma(qv[t], cf, p);
        } else {
          qv[t] = make_double2(0.0, 0.0);
        }
      }
      red[tid] = p;
      __syncthreads();
      if (warp == 0) {
        double2 tot = red[lane];
#pragma unroll
        for (int w = 1; w < PT / 32; ++w) tot = cadd(tot, red[w * 32 + lane]);
        const double2 v = csub(Vb[lane], tot);
        Vb[lane] = v;
        vec[(int64_t)c0 * RB + lane] = v;
      }
      __syncthreads();
      const double2 v = Vb[lane];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        acc[t] = cfmaconj(qv[t], v, acc[t]);
      }
    } else if (PASS != PASS_A) {
      for (int cr = 0; cr < nc; cr += 8) {
        const int nr = min(8, nc - cr);
        const int SL = pass_slices(nr);
        const int cl = warp / SL, sl = warp % SL;
        double2 p = make_double2(0.0, 0.0);
        if (cl < nr) {
          const double2* S = st + (cr + cl) * belem + lane;
#pragma unroll 4
          for (int j = sl; j < J; j += SL) {
            const double2 q = S[j * RB], cf = coef[j];
            p = cfma(q, cf, p);
          }
        }
        red[tid] = p;
        __syncthreads();
        if (sl == 0 && cl < nr) {
          double2 tot = p;
          for (int q = 1; q < SL; ++q) tot = cadd(tot, red[tid + 32 * q]);
          const int c = cr + cl;
          const double2 v = PASS == PASS_X ? cadd(Vb[c * RB + lane], tot) : csub(Vb[c * RB + lane], tot);
          Vb[c * RB + lane] = v;
          const int64_t row = (int64_t)(c0 + c) * RB + lane;
          if (PASS == PASS_C) {
            qblock(a, b, c0 + c)[(size_t)(k + 1) * RB + lane] = v;   // raw q_{k+1}
            a.P[(size_t)row * a.pstride + b] = v;
            nrm += cabs2(v);
          } else {
            vec[row] = v;
          }
        }
        __syncthreads();
      }
    }
    if (PASS == PASS_A) {
      for (int c = 0; c < nc; ++c) {
        const double2* S = st + c * belem + lane;
        const double2 v = Vb[c * RB + lane];
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int j = warp + 8 * t;
          if (j < J) {
            const double2 q = S[j * RB];
            acc[t] = cfmaconj(q, v, acc[t]);
          }
        }
      }
    }
    fence_proxy_async();   // generic-proxy smem writes before the async proxy refills this stage
    __syncthreads();
  }
  if (a.fused && tid < PASS_MAX_STAGES) mbar_inval(&mbar[tid]);   // re-initialised by the next work item
  if (tid == 0 && blk_begin * RB < a.n) {
    // algorithmic bytes of this CTA: J basis rows read + vector read (+ vector/basis row written)
    const int64_t real_rows = min((int64_t)blk_end * RB, (int64_t)a.n) - (int64_t)blk_begin * RB;
    atomicAdd(a.bytes + PASS, (unsigned long long)((J + (PASS == PASS_A ? 1 : 2)) * real_rows * 16));
  }
  if (PASS == PASS_A || PASS == PASS_B) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int j = warp + 8 * t;
      const double x = warp_sum(acc[t].x), y = warp_sum(acc[t].y);
      if (lane == 0 && j < J) part[j] = make_double2(x, y);
    }
  } else if (PASS == PASS_C) {
    red[tid] = make_double2(nrm, 0.0);
    __syncthreads();
    for (int o = PT / 2; o > 0; o >>= 1) {
      if (tid < o) red[tid].x += red[tid + o].x;
      __syncthreads();
    }
    if (tid == 0) part[0] = red[0];
  }
}

// Basis pass for restart > WIDE_RESTART (any J): the same two phases as stream_segment, reading the
// basis straight from global memory (lanes = rows of a 32-row block, coalesced 512-B rows; warps
// split the columns) instead of through the shared-memory ring, whose stage must hold a whole
// J x 32 block.  Dots are taken in tiles of 256 columns (32 register accumulators per thread).
// Coefficients come from global memory: B/C: qs_j * C{1,2}_j, X: Y_j.
template <int PASS>
__device__ __forceinline__ void stream_segment_wide(const KArgs& a, int b, int s, int J, int k, double2* red,
                                                    double2* part) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int segb = a.seg_rows / RB;
  const int blk_begin = s * segb;
  const int blk_end = min(blk_begin + segb, a.nblk);
  double2* vec = (PASS == PASS_X ? a.X : a.W) + (size_t)b * a.ld;
  const double* qs = a.qs + (size_t)b * a.jcap;
  const double2* cc = (PASS == PASS_B ? a.C1 : PASS == PASS_C ? a.C2 : a.Y) + (size_t)b * a.jcap;
  double nrm = 0.0;
  if (PASS != PASS_A) {
    for (int blk = blk_begin; blk < blk_end; ++blk) {
      const double2* S = qblock(a, b, blk) + lane;
      double2 p = make_double2(0.0, 0.0);
#pragma unroll 4
      for (int j = warp; j < J; j += PT / 32) {
        const double2 q = S[(size_t)j * RB];
        const double2 cf = PASS == PASS_X ? cc[j] : cscale(cc[j], qs[j]);
        p = cfma(q, cf, p);
      }
      red[tid] = p;
      __syncthreads();
      if (warp == 0) {
        double2 tot = red[lane];
#pragma unroll
        for (int w = 1; w < PT / 32; ++w) tot = cadd(tot, red[w * 32 + lane]);
        const int64_t row = (int64_t)blk * RB + lane;
        const double2 v = PASS == PASS_X ? cadd(vec[row], tot) : csub(vec[row], tot);
        if (PASS == PASS_C) {
          qblock(a, b, blk)[(size_t)(k + 1) * RB + lane] = v;   // raw q_{k+1}
          a.P[(size_t)row * a.pstride + b] = v;
          nrm += cabs2(v);
        } else {
          vec[row] = v;
        }
      }
      __syncthreads();
    }
  }
  if (PASS == PASS_A || PASS == PASS_B) {
    for (int j0 = 0; j0 < J; j0 += PT) {
      double2 acc[PT / 8];
#pragma unroll
      for (int t = 0; t < PT / 8; ++t) acc[t] = make_double2(0.0, 0.0);
      for (int blk = blk_begin; blk < blk_end; ++blk) {
        const double2 v = vec[(int64_t)blk * RB + lane];
        const double2* S = qblock(a, b, blk) + lane;
#pragma unroll
        for (int t = 0; t < PT / 8; ++t) {
          const int j = j0 + warp + 8 * t;
          if (j < J) {
            const double2 q = S[(size_t)j * RB];
            acc[t] = cfmaconj(q, v, acc[t]);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < PT / 8; ++t) {
        const int j = j0 + warp + 8 * t;
        const double x = warp_sum(acc[t].x), y = warp_sum(acc[t].y);
        if (lane == 0 && j < J) part[j] = make_double2(x, y);
      }
    }
  }
  if (tid == 0 && blk_begin * RB < a.n) {
    const int64_t real_rows = min((int64_t)blk_end * RB, (int64_t)a.n) - (int64_t)blk_begin * RB;
    atomicAdd(a.bytes + PASS, (unsigned long long)((J + (PASS == PASS_A ? 1 : 2)) * real_rows * 16));
  }
  if (PASS == PASS_C) {
    red[tid] = make_double2(nrm, 0.0);
    __syncthreads();
    for (int o = PT / 2; o > 0; o >>= 1) {
      if (tid < o) red[tid].x += red[tid + o].x;
      __syncthreads();
    }
    if (tid == 0) part[0] = red[0];
  }
}

__device__ __forceinline__ void group_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// Pass B for small J (J <= gthr[2]): G = 1, 2 or 4 warps share a 32-row block (thread (wg, lane)
// owns row `lane`, columns j = wg + G*t) and the CTA's 8/G warp groups work on different blocks
// of a chunk at once.  With G = 8 (stream_segment) every block is a CTA-wide step, which leaves
// small-J chunks latency-bound; here a group needs only its own named barrier (none for G = 1).
// Same two phases as stream_segment<PASS_B>: w -= sum_j q_j c_j, then acc_t += conj(q_j) w, with
// the block's basis values held in registers between them.
template <int G, int T>
__device__ __forceinline__ void stream_segment_bg(const KArgs& a, int b, int s, int J, bool rev, const double2* coef,
                                                  double2* smem, uint64_t* mbar, double2* red, double2* part) {
  constexpr int NG = 8 / G;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / G, wg = warp % G;
  const int segb = a.seg_rows / RB;
  const int blk_begin = s * segb;
  const int blk_end = min(blk_begin + segb, a.nblk);
  const int nblocks = blk_end - blk_begin;
  const int belem = J * RB;
  const int blk_elems = belem + RB;
  // chunks of NG blocks (one per group), up to PASS_MAX_STAGES of them in the ring
  const int CB = min(NG, nblocks);
  const int stage_elems = CB * blk_elems;
  const int NS = max(1, min(PASS_MAX_STAGES, a.smem_elems / stage_elems));
  const int AH = pass_ahead(a, NS, stage_elems);
  const int nchunks = (nblocks + CB - 1) / CB;
  double2* vec = a.W + (size_t)b * a.ld;
  auto stage = [&](int ci) { return smem + (size_t)(ci % NS) * stage_elems; };
  auto load_chunk = [&](int ci) {   // single producer thread
    double2* st = stage(ci);
    const int c0 = blk_begin + (rev ? nchunks - 1 - ci : ci) * CB;
    const int nc = min(CB, blk_end - c0);
    uint64_t* bar = &mbar[ci % NS];
    mbar_expect_tx(bar, (unsigned)(nc * blk_elems * 16));
    for (int c = 0; c < nc; ++c) bulk_g2s(st + c * belem, qblock(a, b, c0 + c), (unsigned)belem * 16u, bar);
    bulk_g2s(st + CB * belem, vec + (size_t)c0 * RB, (unsigned)(nc * RB * 16), bar);
  };
  if (tid < PASS_MAX_STAGES) mbar_init(&mbar[tid], 1);
  fence_mbar_init();
  __syncthreads();
  if (tid == 0)
    for (int ci = 0; ci < AH && ci < nchunks; ++ci) load_chunk(ci);
  double2 acc[T];
#pragma unroll
  for (int t = 0; t < T; ++t) acc[t] = make_double2(0.0, 0.0);
  int bi = 0;
  for (int ci = 0; ci < nchunks; ++ci) {
    if (tid == 0 && ci + AH < nchunks) load_chunk(ci + AH);   // stage of chunk ci+AH-NS <= ci-1 (released)
    mbar_wait(&mbar[ci % NS], (unsigned)((ci / NS) & 1));
    const double2* st = stage(ci);
    const int c0 = blk_begin + (rev ? nchunks - 1 - ci : ci) * CB;
    const int nc = min(CB, blk_end - c0);
    const double2* Vb = st + CB * belem;
    if (grp < nc) {
      const int c = grp;
      const double2* S = st + c * belem + lane;
      double2 qv[T];
      double2 p = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = wg + G * t;
        if (j < J) {
          qv[t] = S[j * RB];
          const double2 cf = coef[j];
          p = cfma(qv[t], cf, p);
        } else {
          qv[t] = make_double2(0.0, 0.0);
        }
      }
      const int64_t row = (int64_t)(c0 + c) * RB + lane;
      double2 v;
      if (G == 1) {
        v = csub(Vb[c * RB + lane], p);
        vec[row] = v;
      } else {
        double2* rb = red + (bi & 1) * PT + grp * G * 32;   // group slot, double-buffered
        rb[wg * 32 + lane] = p;
        group_sync(1 + grp, 32 * G);
        if (wg == 0) {
          double2 tot = p;
#pragma unroll
          for (int w = 1; w < G; ++w) tot = cadd(tot, rb[w * 32 + lane]);
          v = csub(Vb[c * RB + lane], tot);
          vec[row] = v;
          rb[lane] = v;
        }
        group_sync(1 + grp, 32 * G);
        v = rb[lane];
      }
#pragma unroll
      for (int t = 0; t < T; ++t) {
        acc[t] = cfmaconj(qv[t], v, acc[t]);
      }
      ++bi;
    }
    fence_proxy_async();
    __syncthreads();
  }
  if (a.fused && tid < PASS_MAX_STAGES) mbar_inval(&mbar[tid]);   // re-initialised by the next work item
  if (tid == 0 && blk_begin * RB < a.n) {
    const int64_t real_rows = min((int64_t)blk_end * RB, (int64_t)a.n) - (int64_t)blk_begin * RB;
    atomicAdd(a.bytes + PASS_B, (unsigned long long)((J + 2) * real_rows * 16));
  }
  // rows -> lanes (warp sums), then groups in fixed order
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const int j = wg + G * t;
    const double x = warp_sum(acc[t].x), y = warp_sum(acc[t].y);
    if (lane == 0 && j < J) red[grp * J + j] = make_double2(x, y);
  }
  __syncthreads();
  for (int j = tid; j < J; j += PT) {
    double2 tot = red[j];
#pragma unroll
    for (int g = 1; g < NG; ++g) tot = cadd(tot, red[g * J + j]);
    part[j] = tot;
  }
}

// One (mode, segment) work item vb of a basis pass (a kernel launch: blockIdx.x; the fused
// persistent kernel: its CTAs walk the work items).  Shared buffers are passed in (the fused kernel
// declares them once); coef doubles as the back-substitution vector y of pass C.
template <int PASS>
__device__ __forceinline__ void pass_body(const KArgs& a, int vb, double2* smem, double2* coef, double2* red,
                                          uint64_t* mbar, int* sflag_, int* s_solve_) {
  int& sflag = *sflag_;
  int& s_solve = *s_solve_;
  double2* ys = coef;
  if (a.fused) {                  // shared buffers of the previous work item / phase
    fence_proxy_async();          // generic smem writes (pass C staging) before the next bulk copies
    __syncthreads();
  }
  const int b = vb % a.nb, s = vb / a.nb;
  ModeCtl* c = a.ctl + b;
  const int phase = c->phase;
  const int tid = threadIdx.x;
  if (PASS == PASS_A && phase == PH_XUPDATE && a.x_in_a) {
    // cycle-end x += Q y rides on the next tick's pass-A launch (one launch per tick saved)
    const int kx = c->k;
    if (a.wide) {
      stream_segment_wide<PASS_X>(a, b, s, kx, kx, red, nullptr);
    } else {
      for (int j = tid; j < kx; j += PT) coef[j] = a.Y[(size_t)b * a.jcap + j];
      __syncthreads();
      stream_segment<PASS_X, 1>(a, b, s, kx, kx, coef, smem, mbar, red, nullptr);
    }
    if (!last_cta(a, b, PASS_X, a.nseg, &sflag)) return;
    if (tid == 0) c->phase = PH_RESID;
    return;
  }
  if (PASS == PASS_X ? phase != PH_XUPDATE : phase != PH_INNER) return;
  const int k = c->k;
  const int J = PASS == PASS_X ? k : k + 1;
  double* qs = a.qs + (size_t)b * a.jcap;
  double2* part = a.part + (size_t)b * a.nseg * a.jcap + (size_t)s * a.jcap;
  const int T = (J + 7) / 8;
  // Streaming direction (SS_PASS_ALT): A and C forward on even k, B the other way, all flipped on
  // odd k, so every pass starts on the rows its predecessor read last (still in L2 when the
  // batch's basis is not much larger than L2).  Depends only on this mode's k: batch-invariant.
  const bool rev = a.pass_alt && (((k & 1) != 0) != (PASS == PASS_B));
  if (a.wide) {
    stream_segment_wide<PASS>(a, b, s, J, k, red, part);
  } else {
  // coefficients of the update (qs folded in): B: qs_j c_j, C: qs_j c2_j, X: y_j (already scaled)
  if (PASS == PASS_B || PASS == PASS_C) {
    const double2* cc = (PASS == PASS_B ? a.C1 : a.C2) + (size_t)b * a.jcap;
    for (int j = tid; j < J; j += PT) coef[j] = cscale(cc[j], qs[j]);
  } else if (PASS == PASS_X) {
    for (int j = tid; j < J; j += PT) coef[j] = a.Y[(size_t)b * a.jcap + j];
  }
  __syncthreads();
  if (PASS == PASS_B && J <= a.gthr[2]) {
    if (J <= a.gthr[0]) {
      if (J <= 4) stream_segment_bg<1, 4>(a, b, s, J, rev, coef, smem, mbar, red, part);
      else if (J <= 8) stream_segment_bg<1, 8>(a, b, s, J, rev, coef, smem, mbar, red, part);
      else stream_segment_bg<1, 16>(a, b, s, J, rev, coef, smem, mbar, red, part);
    } else if (J <= a.gthr[1]) {
      stream_segment_bg<2, 16>(a, b, s, J, rev, coef, smem, mbar, red, part);
    } else {
      stream_segment_bg<4, 16>(a, b, s, J, rev, coef, smem, mbar, red, part);
    }
  } else if (PASS == PASS_A || PASS == PASS_B) {
    if (T <= 2) stream_segment<PASS, 2>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
    else if (T <= 4) stream_segment<PASS, 4>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
    else if (T <= 8) stream_segment<PASS, 8>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
    else if (T <= 16) stream_segment<PASS, 16>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
    else if (T <= 26) stream_segment<PASS, 26>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
    else stream_segment<PASS, 32>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
  } else {
    stream_segment<PASS, 1>(a, b, s, J, k, coef, smem, mbar, red, part, rev);
  }
  }   // !a.wide
  if (PASS == PASS_X) {
    if (!last_cta(a, b, PASS, a.nseg, &sflag)) return;
    if (tid == 0) c->phase = PH_RESID;
    return;
  }
  if (!last_cta(a, b, PASS, a.nseg, &sflag)) return;

  // ---- last CTA of this mode: reduce partials over segments in fixed order ----
  const double2* pb = a.part + (size_t)b * a.nseg * a.jcap;
  const int JA = PASS == PASS_C ? 1 : J;
  int SL = 1;
  for (int jb = 0; jb < JA; jb += PT) {   // one tile unless J > 256 (wide restart)
  const int JR = min(PT, JA - jb);
  SL = max(1, PT / JR);      // slices over segments
  {
    // 8 independent accumulators keep 8 L2 loads in flight per thread; combined in fixed order
    const int j = jb + tid % JR, sl = tid / JR;
    double2 acc8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc8[u] = make_double2(0.0, 0.0);
    if (sl < SL) {
      int q = sl;
      for (; q + 7 * SL < a.nseg; q += 8 * SL) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(pb + (size_t)(q + u * SL) * a.jcap + j);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc8[u] = cadd(acc8[u], v[u]);
      }
      for (int u = 0; q < a.nseg; q += SL, ++u) acc8[u] = cadd(acc8[u], __ldcg(pb + (size_t)q * a.jcap + j));
    }
    double2 acc = acc8[0];
#pragma unroll
    for (int u = 1; u < 8; ++u) acc = cadd(acc, acc8[u]);
    red[tid] = acc;
  }
  __syncthreads();
  if (PASS == PASS_A || PASS == PASS_B) {
    double2* out = (PASS == PASS_A ? a.C1 : a.C2) + (size_t)b * a.jcap;
    if (tid < JR) {
      double2 acc = red[tid];
      for (int q = 1; q < SL; ++q) acc = cadd(acc, red[q * JR + tid]);
      out[jb + tid] = cscale(acc, qs[jb + tid]);
    }
    __syncthreads();
  }
  }
  if (PASS == PASS_A || PASS == PASS_B) return;
  // PASS_C: Givens update (krylov.py:115-149).  The H column and the stored rotations are staged
  // in (now idle) shared memory by all threads; one thread runs the serial recurrence on them.
  const int jc = a.jcap;
  // wide restart: the column, rotations and y live in global memory (H column k, CS, SN, Y)
  double2* hcol = a.H + ((size_t)b * a.restart + k) * jc;      // column k, rows 0..restart
  double2* hs = a.wide ? hcol : smem;                           // column k (k+2 entries)
  const double2* css = a.wide ? a.CS + (size_t)b * a.restart : smem + 256;   // cs[0..k)
  const double2* sns = a.wide ? a.SN + (size_t)b * a.restart : smem + 512;   // sn[0..k)
  double2* y = a.wide ? a.Y + (size_t)b * jc : ys;
  {
    const double2* c1 = a.C1 + (size_t)b * jc;
    const double2* c2 = a.C2 + (size_t)b * jc;
    const double2* csg = a.CS + (size_t)b * a.restart;
    const double2* sng = a.SN + (size_t)b * a.restart;
    for (int i = tid; i <= k; i += PT) {
      hs[i] = cadd(c1[i], c2[i]);
      if (i < k && !a.wide) { smem[256 + i] = csg[i]; smem[512 + i] = sng[i]; }
    }
  }
  __syncthreads();
  if (tid == 0) {
    double nsq = 0;
    for (int q = 0; q < SL; ++q) nsq += red[q].x;
    const double hk = sqrt(nsq);
    double2* h = hs;
    double2* cs = a.CS + (size_t)b * a.restart;
    double2* sn = a.SN + (size_t)b * a.restart;
    double2* g = a.G + (size_t)b * jc;
    double2 hi = h[0];
    for (int i = 0; i < k; ++i) {
      const double2 hi1 = h[i + 1], ci = css[i], si = sns[i];
      h[i] = cadd(cmul(ci, hi), cmul(si, hi1));
      hi = cadd(cmul(make_double2(-si.x, si.y), hi), cmul(conjd(ci), hi1));
    }
    h[k] = hi;
    const double ahkk = hypot(h[k].x, h[k].y);
    const double denom = sqrt(ahkk * ahkk + hk * hk);
    int exit_cycle = 0;
    if (denom == 0.0) {                       // krylov.py:124-129
      c->breakdown = 1;
      c->iters += 1;
      exit_cycle = 1;
    } else {
      const double2 csk = cscale(conjd(h[k]), 1.0 / denom);
      const double2 snk = make_double2(hk / denom, 0.0);
      cs[k] = csk;
      sn[k] = snk;
      h[k] = cadd(cmul(csk, h[k]), cscale(snk, hk));
      const double2 gk = g[k];
      g[k + 1] = cmul(make_double2(-snk.x, snk.y), gk);
      g[k] = cmul(csk, gk);
      c->iters += 1;
      const double est = hypot(g[k + 1].x, g[k + 1].y);
      c->est = est;
      if (c->hist_len < a.hist_cap) a.hist[(size_t)b * a.hist_cap + c->hist_len] = est;
      c->hist_len += 1;
      if (hk <= 1e-14 * fabs(c->beta)) {      // happy breakdown (krylov.py:141-145)
        c->breakdown = 1;
        c->k = k + 1;
        exit_cycle = 1;
      } else {
        qs[k + 1] = 1.0 / hk;
        c->k = k + 1;
        if (est <= c->target || c->k >= a.restart || c->iters >= c->maxiter) exit_cycle = 1;
      }
    }
    h[k + 1] = make_double2(hk, 0.0);
    if (denom != 0.0) h[k + 1] = make_double2(0.0, 0.0);
    s_solve = 0;
    if (exit_cycle) {
      const int kk = c->k;
      c->gk_last = hypot(g[kk].x, g[kk].y);
      if (kk > 0) {
        s_solve = kk;
      } else {
        c->phase = PH_RESID;
      }
    }
  }
  __syncthreads();
  if (!a.wide)
    for (int i = tid; i <= k + 1; i += PT) hcol[i] = hs[i];
  __syncthreads();
  const int kk = s_solve;
  if (kk == 0) return;
  // Cycle end: y = H[:k,:k]^-1 g[:k] (column-oriented back substitution, krylov.py:151-153,167-168)
  const double2* hb = a.H + (size_t)b * a.restart * jc;
  const double2* g = a.G + (size_t)b * jc;
  for (int i = tid; i < kk; i += PT) y[i] = g[i];
  __syncthreads();
  for (int j = kk - 1; j >= 0; --j) {
    if (tid == 0) y[j] = cdiv(y[j], hb[(size_t)j * jc + j]);
    __syncthreads();
    const double2 yj = y[j];
    for (int i = tid; i < j; i += PT) y[i] = csub(y[i], cmul(hb[(size_t)j * jc + i], yj));
    __syncthreads();
  }
  for (int i = tid; i < kk; i += PT) a.Y[(size_t)b * jc + i] = cscale(y[i], qs[i]);   // in place when wide
  __syncthreads();
  if (tid == 0) c->phase = PH_XUPDATE;
}

template <int PASS>
__global__ void __launch_bounds__(PT, 1) k_pass(KArgs a) {
  extern __shared__ __align__(128) double2 smem[];
  __shared__ double2 coef[256];
  __shared__ double2 red[PASS == PASS_B ? 2 * PT : PT];
  __shared__ __align__(8) uint64_t mbar[PASS_MAX_STAGES];
  __shared__ int sflag, s_solve;
  pass_body<PASS>(a, blockIdx.x, smem, coef, red, mbar, &sflag, &s_solve);
}

// ------------------------------------------------------------------------------------------------
// Persistent fused tick (small n): ONE cooperative launch runs `nticks` ticks; its CTAs (one per
// SM) walk the virtual blocks of the tick SpMV and the (mode, segment) work items of passes A, B, C
// with a grid barrier between phases -- the same work decomposition, reduction trees and last-CTA
// state changes as the four-kernel tick, so per-mode results are bitwise identical to it, without
// four kernel launches, four ring fills from a cold start and four launch tails per tick.
// Memory ordering across phases: the barrier is a gpu-scope fence + arrive/wait (cooperative
// groups); generic-proxy global writes (W, Q, P, X) are ordered before the next phase's bulk copies
// by fence.proxy.async on both sides; x-type vectors written in the launch are never read through
// the non-coherent path (NC = false).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void fused_sync(cg::grid_group& grid) {
  asm volatile("fence.proxy.async;\n" ::: "memory");
  grid.sync();
  asm volatile("fence.proxy.async;\n" ::: "memory");
}

template <int DIM>
__global__ void __launch_bounds__(PT, 1) k_tick_fused(KArgs a, int nticks, int tick0) {
  extern __shared__ __align__(128) double2 smem[];
  __shared__ double2 coef[256];
  __shared__ double2 red[2 * PT];
  __shared__ __align__(8) uint64_t mbar[PASS_MAX_STAGES];
  __shared__ int sph[MAXB_SMEM];
  __shared__ int sflag, s_any, s_solve;
  // SpMV-phase mode state lives in the upper half of red (the finalize reduction uses the lower
  // half), so the basis-pass ring keeps the four-kernel tick's size: same chunking, same sums
  double* som = (double*)(red + PT);
  double* sxs = som + MAXB_SMEM;
  cg::grid_group grid = cg::this_grid();
  const int nspmv = a.nsb * a.spmv_split, npass = a.nb * a.nseg;
  auto stamp = [&](int t, int q) {   // optional phase timestamps (SS_FUSED_PROF)
    if (a.ptime && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      a.ptime[(size_t)(t % FUSED_PROF_TICKS) * 5 + q] = (long long)g;
    }
  };
  for (int t = 0; t < nticks; ++t) {
    const int tt = tick0 + t;
    stamp(tt, 0);
    for (int vb = blockIdx.x; vb < nspmv; vb += gridDim.x)
      tick_spmv_body<DIM, 0, false>(a, vb, nspmv, sph, som, sxs, &sflag, &s_any, red);
    fused_sync(grid);
    stamp(tt, 1);
    // n_done only changes in the SpMV phase: every CTA reads the same value here
    const bool stop = *(volatile int*)a.n_done >= a.nb;
    for (int vb = blockIdx.x; vb < npass; vb += gridDim.x) pass_body<PASS_A>(a, vb, smem, coef, red, mbar, &sflag, &s_solve);
    fused_sync(grid);
    stamp(tt, 2);
    for (int vb = blockIdx.x; vb < npass; vb += gridDim.x) pass_body<PASS_B>(a, vb, smem, coef, red, mbar, &sflag, &s_solve);
    fused_sync(grid);
    stamp(tt, 3);
    for (int vb = blockIdx.x; vb < npass; vb += gridDim.x) pass_body<PASS_C>(a, vb, smem, coef, red, mbar, &sflag, &s_solve);
    fused_sync(grid);
    stamp(tt, 4);
    if (stop) break;
  }
}

__global__ void k_finalize(KArgs a) {
  const int b = blockIdx.y;
  if (b >= a.nb || !a.ctl[b].zero_x) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.ld; i += (int64_t)gridDim.x * blockDim.x)
    a.X[(size_t)b * a.ld + i] = make_double2(0.0, 0.0);
}

// Jacobi scale of a generic CSR matrix: 1/diag, 1 where the diagonal is zero or absent (krylov.py:49-60).
__global__ void k_csr_jacobi(SsCsrDev A, double2* __restrict__ out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int set = blockIdx.y;
  if (row >= A.n) return;
  double2 d = make_double2(0.0, 0.0);
  for (int e = A.indptr[row]; e < A.indptr[row + 1]; ++e)
    if (A.indices[e] == row) d = cadd(d, A.vals[(size_t)set * A.nnz + e]);
  out[(size_t)set * A.n + row] = (d.x == 0.0 && d.y == 0.0) ? make_double2(1.0, 0.0) : cdiv(make_double2(1.0, 0.0), d);
}

// True residual partials: spart[b][blk] = (||b - A x||^2, ||b||^2) over the block's rows
// (ComplexSaddleSystem.residual_norm, assembly.py:357-362; gmres_solve, krylov.py:203-207).
template <int DIM>
__global__ void __launch_bounds__(PT) k_true_resid(KArgs a) {
  __shared__ double red[2][PT / 32];
  const int b = blockIdx.x % a.nb, sb = blockIdx.x / a.nb;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double om = a.ctl[b].omega;
  const double2* x = a.X + (size_t)b * a.ld;
  const double2* rhs = a.RHS + (size_t)b * a.ld;
  double tt = 0, bb = 0;
  auto emit = [&](int row, double2 v) {
    const double2 rb = rhs[row];
    tt += cabs2(csub(rb, v));
    bb += cabs2(rb);
  };
  if (a.kind == 0) saddle_block<DIM>(a.op, sb, om, x, emit);
  else csr_block(a.csr, a.csr.nvals > 1 ? b : 0, sb, x, emit);
  tt = warp_sum(tt);
  bb = warp_sum(bb);
  if (lane == 0) { red[0][warp] = tt; red[1][warp] = bb; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0, s1 = 0;
    for (int w = 0; w < PT / 32; ++w) { s0 += red[0][w]; s1 += red[1][w]; }
    a.spart[(size_t)b * a.nsb + sb] = make_double2(s0, s1);
  }
}

// ------------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------------
struct ss_krylov {
  int device = 0;
  KArgs a{};
  int max_batch = 0;
  std::vector<void*> allocs;
  cudaStream_t cap_stream = nullptr;
  std::map<int64_t, cudaGraphExec_t> graphs;
  int* h_done = nullptr;       // pinned
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int ticks_per_graph = 8;
  int device_loop = 0;         // whole solve as one graph with a conditional WHILE node (SS_DEVICE_LOOP=0: host-polled)
  size_t smem_pass = 0;
  int64_t last_ticks = 0;
  int64_t last_launches = 0;
  double2* csr_vals_owned = nullptr;
  int stream_ctas = 2 * 148;   // persistent CTAs of the staged tick SpMV (2 per SM)
  int row_ctas = 16 * 148;     // grid-stride CTAs of the row-layout tick SpMV
  int fused = 0;               // persistent fused tick kernel (option "fused"; default for small n)
  int fused_grid = 0;          // its CTAs (one per SM), 0 = not set up yet, -1 = unavailable
  int fused_elems = 0;         // its basis-pass ring (double2 elements)
  long long* ptime = nullptr;  // fused phase timestamps (SS_FUSED_PROF=path: written per solve)
};

template <class T>
static int kalloc(ss_krylov* K, size_t count, T** p) {
  SS_CUDA(cudaMalloc((void**)p, std::max<size_t>(1, count) * sizeof(T)));
  K->allocs.push_back((void*)*p);
  SS_CUDA(cudaMemset(*p, 0, std::max<size_t>(1, count) * sizeof(T)));
  return SS_OK;
}

static int krylov_common_init(ss_krylov* K, int n, int max_batch, int restart, int64_t hist_cap) {
  if (restart < 1 || restart > (1 << 20)) { ss_set_error("restart must lie in [1, 2^20]"); return SS_ERR_ARG; }
  if (max_batch < 1 || max_batch > MAXB_SMEM) { ss_set_error("max_batch must lie in [1, 256]"); return SS_ERR_ARG; }
  KArgs& a = K->a;
  a.n = n;
  a.ld = ss_round_up(std::max(n, 1), RB);
  a.nblk = (int)(a.ld / RB);
  a.restart = restart;
  a.jcap = restart + 1;
  a.hist_cap = std::max<int64_t>(1, hist_cap);
  // segment rows depend on n only (batch-composition invariance of every reduction): ~16 segments
  // for small n (config 1: one wave of CTAs for 9 modes, +25 %), 6144 rows for large n (config 2:
  // 2 210 CTAs = 14.9 waves of 148 for 17 modes; 4096 and 8192 measured 1 % slower)
  // 2D saddle systems: ~24 segments (config 1 through the concurrent sub-batches: 14.96 vs 13.82
  // modes/s; 3D at the same n -- pipe3d -- stays best at 16: 5.11 vs 4.96).  A rule on the system
  // (n, dim), never on the batch, so per-mode results stay batch-invariant.
  int64_t segdiv = (K->a.kind == 0 && K->a.op.dim == 2) ? 24 : 16, segmin = 256, segmax = 6144;
  if (const char* e = getenv("SS_SEG_DIV")) segdiv = std::max(1, atoi(e));
  if (const char* e = getenv("SS_SEG_MIN")) segmin = std::max(32, atoi(e));
  if (const char* e = getenv("SS_SEG_MAX")) segmax = std::max(64, atoi(e));
  int64_t seg = ss_round_up((a.ld + segdiv - 1) / segdiv, 32);
  seg = std::min<int64_t>(segmax, std::max<int64_t>(segmin, seg));
  a.seg_rows = (int)seg;
  a.nseg = (int)((a.ld + seg - 1) / seg);
  a.smem_elems = PASS_SMEM_ELEMS;
  a.stage_div = 0;   // 0 = per-pass default
  if (const char* e = getenv("SS_PASS_SMEM")) a.smem_elems = std::max(2048, std::min(PASS_SMEM_ELEMS, atoi(e)));
  a.wide = restart > WIDE_RESTART ? 1 : 0;
  if (!a.wide) a.smem_elems = std::max(a.smem_elems, a.jcap * RB + 2 * RB);   // one full-J block + vector must fit a stage
  else a.smem_elems = 3 * 256;                                                  // no ring; pass C staging unused
  if (const char* e = getenv("SS_PASS_DIV")) a.stage_div = std::max(1, atoi(e));
  a.ahead_bytes = 0;
  if (const char* e = getenv("SS_PASS_AHEAD")) a.ahead_bytes = std::max(0, atoi(e));
  a.pass_alt = 0;
  if (const char* e = getenv("SS_PASS_ALT")) a.pass_alt = atoi(e) != 0;
  K->max_batch = max_batch;
  const size_t B = max_batch;
  int rc;
  if ((rc = kalloc(K, B * a.jcap * a.ld, &a.Q))) return rc;
  if ((rc = kalloc(K, B * a.ld, &a.W))) return rc;
  if ((rc = kalloc(K, B * a.ld, &a.P))) return rc;
  a.pstride = max_batch;
  if (a.spmv_split < 1) a.spmv_split = 1;   // the saddle creator sets it from nsb
  if ((rc = kalloc(K, B * a.ld, &a.X))) return rc;
  if ((rc = kalloc(K, B * a.ld, &a.RHS))) return rc;
  if ((rc = kalloc(K, B * a.jcap, &a.qs))) return rc;
  if ((rc = kalloc(K, B * restart * a.jcap, &a.H))) return rc;
  if ((rc = kalloc(K, B * a.jcap, &a.G))) return rc;
  if ((rc = kalloc(K, B * restart, &a.CS))) return rc;
  if ((rc = kalloc(K, B * restart, &a.SN))) return rc;
  if ((rc = kalloc(K, B * a.jcap, &a.C1))) return rc;
  if ((rc = kalloc(K, B * a.jcap, &a.C2))) return rc;
  if ((rc = kalloc(K, B * a.jcap, &a.Y))) return rc;
  if ((rc = kalloc(K, B * a.nseg * a.jcap, &a.part))) return rc;
  if ((rc = kalloc(K, B * 8, &a.counters))) return rc;
  if ((rc = kalloc(K, 1, &a.n_done))) return rc;
  if ((rc = kalloc(K, B, &a.ctl))) return rc;
  if ((rc = kalloc(K, B * a.hist_cap, &a.hist))) return rc;
  if ((rc = kalloc(K, 8, &a.bytes))) return rc;
  if ((rc = kalloc(K, 3, &a.loop))) return rc;
  SS_CUDA(cudaHostAlloc((void**)&K->h_done, 2 * sizeof(int), cudaHostAllocDefault));
  SS_CUDA(cudaStreamCreateWithFlags(&K->cap_stream, cudaStreamNonBlocking));
  SS_CUDA(cudaEventCreateWithFlags(&K->ev[0], cudaEventDisableTiming));
  SS_CUDA(cudaEventCreateWithFlags(&K->ev[1], cudaEventDisableTiming));
  K->smem_pass = (size_t)a.smem_elems * sizeof(double2);
  if (K->smem_pass + 3 * 256 * sizeof(double2) + 64 > 227 * 1024) {
    ss_set_error("restart too large for the shared-memory staging of the basis passes");
    return SS_ERR_ARG;
  }
  auto setattr = [&](const void* f) {   // per-function attribute: the largest any workspace may request
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(PASS_SMEM_ELEMS * sizeof(double2)));
  };
  SS_CUDA(setattr((const void*)k_pass<PASS_A>));
  SS_CUDA(setattr((const void*)k_pass<PASS_B>));
  SS_CUDA(setattr((const void*)k_pass<PASS_C>));
  SS_CUDA(setattr((const void*)k_pass<PASS_X>));
  SS_CUDA(cudaFuncSetAttribute((const void*)k_tick_spmv_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, STREAM_SMEM));
  SS_CUDA(cudaFuncSetAttribute((const void*)k_tick_spmv_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, STREAM_SMEM));
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    K->stream_ctas = 2 * sms;
    K->row_ctas = 16 * sms;
    if (const char* e = getenv("SS_ROW_CTAS")) K->row_ctas = std::max(1, atoi(e));
    // row blocks dealt in order from an atomic counter: the blocks in flight stay one compact
    // window of the matrix stream and the CTAs stay balanced (config 5: 3.72 vs 3.83 ms in-cycle,
    // same box; results bitwise identical -- blocks and their sums do not change)
    K->a.row_dyn = 1;
    if (const char* e = getenv("SS_ROW_DYN")) K->a.row_dyn = atoi(e);

    if (const char* e = getenv("SS_STREAM_CTAS")) K->stream_ctas = std::max(1, atoi(e));
    K->a.stream_spmv = 0;   // measured slower than the per-block row kernel at config 5
    if (const char* e = getenv("SS_SPMV_STREAM")) K->a.stream_spmv = atoi(e);
  }
  K->ticks_per_graph = n < 200000 ? 16 : 2;
  // persistent fused tick for small systems, where the four tick kernels are launch/latency bound
  K->fused = 0;
  if (const char* e = getenv("SS_FUSED")) K->fused = atoi(e);
  if (getenv("SS_FUSED_PROF")) {
    int rc2 = kalloc(K, (size_t)FUSED_PROF_TICKS * 5, &K->ptime);
    if (rc2) return rc2;
  }
  if (const char* e = getenv("SS_DEVICE_LOOP")) K->device_loop = atoi(e);
  K->a.x_in_a = 1;
  // pass-B grouped mapping thresholds (a rule on n only): small systems switch to wider groups
  // earlier (pipe3d 5.34 vs 5.15 modes/s, config 1 +1 %); large ones keep narrow groups longer
  // (config 5 pass B at J <= 70: 6 216 vs 5 022 GB/s with the small-n thresholds)
  const bool small_n = n < 200000;
  K->a.gthr[0] = small_n ? 8 : 16;
  K->a.gthr[1] = small_n ? 16 : 32;
  K->a.gthr[2] = small_n ? 32 : 64;
  if (const char* e = getenv("SS_PASS_G")) sscanf(e, "%d,%d,%d", &K->a.gthr[0], &K->a.gthr[1], &K->a.gthr[2]);
  // T <= 16 columns per thread below G = 8 (register budget)
  K->a.gthr[0] = std::min(K->a.gthr[0], 16);
  K->a.gthr[1] = std::min(K->a.gthr[1], 32);
  K->a.gthr[2] = std::min(K->a.gthr[2], 64);
  if (const char* e = getenv("SS_X_IN_A")) K->a.x_in_a = atoi(e);
  if (const char* e = getenv("SS_TICKS_PER_GRAPH")) K->ticks_per_graph = std::max(1, atoi(e));
  return SS_OK;
}

extern "C" int ss_krylov_create_saddle(const ss_pattern* P, int max_batch, int restart, int64_t hist_cap,
                                       ss_krylov** out) {
  if (!P || !out) { ss_set_error("null argument"); return SS_ERR_ARG; }
  if (!P->assembled) { ss_set_error("pattern not assembled"); return SS_ERR_STATE; }
  SS_CUDA(cudaSetDevice(P->device));
  ss_krylov* K = new ss_krylov();
  K->device = P->device;
  K->a.kind = 0;
  K->a.op = P->op;
  K->a.nsb = saddle_nsb_host(P->nfree, P->npf);
  {
    // row-layout INNER SpMV from 25 M DOFs up (config 5: one mode per GPU at restart 200, where
    // one lane per row starves the gathers: SpMV -21 %, cycle +5 %; at two modes (config 4) the
    // interleaved kernel stays ahead).  A rule on n only keeps per-mode results batch-invariant.
    int64_t thr = 25000000;
    if (const char* e = getenv("SS_ROW_SPMV_N")) thr = atoll(e);
    K->a.row_spmv = P->op.n >= thr ? 1 : 0;
  }
  // sub-CTAs per SpMV row block when there are few blocks: about two (row, mode) pairs of a
  // 128-row block per thread, and no more than needed to fill the GPU (config 1: 9)
  K->a.spmv_split = std::max(1, std::min(std::min(16, (8 * 148 + K->a.nsb - 1) / K->a.nsb),
                                         (SPMV_VROWS * max_batch + PT / 2 - 1) / (PT / 2)));
  if (const char* e = getenv("SS_SPMV_SPLIT")) K->a.spmv_split = std::max(1, atoi(e));
  int rc = krylov_common_init(K, P->op.n, max_batch, restart, hist_cap);
  if (!rc) rc = kalloc(K, (size_t)max_batch * K->a.nsb, &K->a.spart);
  if (rc) { delete K; return rc; }
  *out = K;
  return SS_OK;
}

// Generic CSR operator: values for nvals sets (1 = shared); scale (optional) per set.
extern "C" int ss_krylov_create_csr(int device, int n, int64_t nnz, const int32_t* indptr, const int32_t* indices,
                                    int nvals, const double* vals, const double* scale, int jacobi_from_diag,
                                    int max_batch, int restart, int64_t hist_cap, ss_krylov** out) {
  if (!out || n <= 0 || !indptr || (nnz > 0 && (!indices || !vals)) || nvals < 1) {
    ss_set_error("bad arguments");
    return SS_ERR_ARG;
  }
  SS_CUDA(cudaSetDevice(device));
  ss_krylov* K = new ss_krylov();
  K->device = device;
  K->a.kind = 1;
  SsCsrDev& A = K->a.csr;
  A.n = n;
  A.nnz = nnz;
  A.nvals = nvals;
  int rc = SS_OK;
  int *ip, *ix;
  double2 *v, *sc = nullptr;
  if (!rc) rc = kalloc(K, (size_t)n + 1, &ip);
  if (!rc) rc = kalloc(K, (size_t)nnz, &ix);
  if (!rc) rc = kalloc(K, (size_t)nvals * nnz, &v);
  if (!rc && (scale || jacobi_from_diag)) rc = kalloc(K, (size_t)nvals * n, &sc);
  if (rc) { delete K; return rc; }
  SS_CUDA(cudaMemcpy(ip, indptr, sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
  if (nnz) SS_CUDA(cudaMemcpy(ix, indices, sizeof(int) * nnz, cudaMemcpyHostToDevice));
  if (nnz) SS_CUDA(cudaMemcpy(v, vals, sizeof(double2) * nvals * nnz, cudaMemcpyHostToDevice));
  if (scale) SS_CUDA(cudaMemcpy(sc, scale, sizeof(double2) * nvals * n, cudaMemcpyHostToDevice));
  A.indptr = ip; A.indices = ix; A.vals = v; A.scale = sc;
  if (jacobi_from_diag && !scale) {
    k_csr_jacobi<<<dim3((n + 255) / 256, nvals), 256>>>(A, sc);
    ss_count_launch();
    SS_CUDA(cudaGetLastError());
  }
  K->a.nsb = (n + SPMV_PROWS - 1) / SPMV_PROWS;
  rc = krylov_common_init(K, n, max_batch, restart, hist_cap);
  if (!rc) rc = kalloc(K, (size_t)max_batch * K->a.nsb, &K->a.spart);
  if (rc) { delete K; return rc; }
  *out = K;
  return SS_OK;
}

extern "C" void ss_krylov_destroy(ss_krylov* K) {
  if (!K) return;
  cudaSetDevice(K->device);
  for (auto& kv : K->graphs) cudaGraphExecDestroy(kv.second);
  for (void* p : K->allocs) cudaFree(p);
  if (K->h_done) cudaFreeHost(K->h_done);
  if (K->cap_stream) cudaStreamDestroy(K->cap_stream);
  for (auto e : K->ev) if (e) cudaEventDestroy(e);
  delete K;
}

// Workspace options (A/B and parity coverage of layout-dependent code paths).  Changing an option
// drops the cached graphs.  "row_spmv": 1 = row-layout tick SpMV (8 lanes per node row, strided P
// column), 0 = mode-interleaved; "device_loop": conditional-WHILE graph; "ticks_per_graph".
extern "C" int ss_krylov_set_option(ss_krylov* K, const char* name, int64_t value) {
  if (!K || !name) { ss_set_error("null argument"); return SS_ERR_ARG; }
  const std::string opt(name);
  if (opt == "row_spmv") {
    if (K->a.kind != 0 && value) { ss_set_error("row_spmv applies to the saddle operator only"); return SS_ERR_ARG; }
    K->a.row_spmv = value ? 1 : 0;
  } else if (opt == "stream_spmv") {
    K->a.stream_spmv = value ? 1 : 0;
  } else if (opt == "device_loop") {
    K->device_loop = value ? 1 : 0;
  } else if (opt == "ticks_per_graph") {
    if (value < 1 || value > 1024) { ss_set_error("ticks_per_graph must lie in [1, 1024]"); return SS_ERR_ARG; }
    K->ticks_per_graph = (int)value;
  } else if (opt == "fused") {
    K->fused = value ? 1 : 0;
  } else if (opt == "pass_alt") {
    K->a.pass_alt = value ? 1 : 0;
  } else {
    ss_set_error("unknown workspace option '" + opt + "'");
    return SS_ERR_ARG;
  }
  SS_CUDA(cudaSetDevice(K->device));
  for (auto& kv : K->graphs) cudaGraphExecDestroy(kv.second);
  K->graphs.clear();
  return SS_OK;
}

extern "C" int ss_krylov_get_option(const ss_krylov* K, const char* name, int64_t* value) {
  if (!K || !name || !value) { ss_set_error("null argument"); return SS_ERR_ARG; }
  const std::string opt(name);
  if (opt == "row_spmv") *value = K->a.row_spmv;
  else if (opt == "stream_spmv") *value = K->a.stream_spmv;
  else if (opt == "device_loop") *value = K->device_loop;
  else if (opt == "ticks_per_graph") *value = K->ticks_per_graph;
  else if (opt == "fused") *value = K->fused;
  else if (opt == "pass_alt") *value = K->a.pass_alt;
  else if (opt == "fused_active") *value = K->fused && !(K->a.kind == 0 && K->a.row_spmv) && K->fused_grid >= 0;
  else { ss_set_error("unknown workspace option '" + opt + "'"); return SS_ERR_ARG; }
  return SS_OK;
}

// info: [n, ld, restart, nseg, seg_rows, nsb, max_batch, ticks_per_graph, smem_pass, kind]
extern "C" int ss_krylov_info(const ss_krylov* K, int64_t* info) {
  if (!K || !info) { ss_set_error("null argument"); return SS_ERR_ARG; }
  info[0] = K->a.n; info[1] = K->a.ld; info[2] = K->a.restart; info[3] = K->a.nseg; info[4] = K->a.seg_rows;
  info[5] = K->a.nsb; info[6] = K->max_batch; info[7] = K->ticks_per_graph; info[8] = (int64_t)K->smem_pass;
  info[9] = K->a.kind;
  return SS_OK;
}

extern "C" int ss_krylov_buffers(ss_krylov* K, double** rhs, double** x, int64_t* ld) {
  if (!K) { ss_set_error("null argument"); return SS_ERR_ARG; }
  if (rhs) *rhs = (double*)K->a.RHS;
  if (x) *x = (double*)K->a.X;
  if (ld) *ld = K->a.ld;
  return SS_OK;
}

template <int DIM>
static void tick_spmv_launch_dims(const ss_krylov* K, const KArgs& a, unsigned* grid, size_t* smem) {
  if (tick_streamed(a)) {
    *grid = (unsigned)std::max(1, std::min(a.op.nchunk, K->stream_ctas));
    *smem = STREAM_SMEM;
  } else if (a.kind == 0 && a.row_spmv) {
    *grid = (unsigned)std::max(1, std::min(a.nsb, K->row_ctas));
    *smem = 0;
  } else {
    *grid = (unsigned)(a.nsb * a.spmv_split);
    *smem = 0;
  }
}

template <int DIM>
static int launch_tick(ss_krylov* K, const KArgs& a, cudaStream_t st) {
  const unsigned gs = (unsigned)(a.nb * a.nseg);
  unsigned sgrid;
  size_t ssmem;
  tick_spmv_launch_dims<DIM>(K, a, &sgrid, &ssmem);
  if (ssmem) k_tick_spmv_stream<DIM><<<sgrid, PT, ssmem, st>>>(a);
  else if (a.kind == 0 && a.row_spmv) k_tick_spmv<DIM, 1><<<sgrid, PT, 0, st>>>(a);
  else k_tick_spmv<DIM, 0><<<sgrid, PT, 0, st>>>(a);
  SS_LAUNCH_CHECK();
  k_pass<PASS_A><<<gs, PT, K->smem_pass, st>>>(a);
  SS_LAUNCH_CHECK();
  k_pass<PASS_B><<<gs, PT, K->smem_pass, st>>>(a);
  SS_LAUNCH_CHECK();
  k_pass<PASS_C><<<gs, PT, K->smem_pass, st>>>(a);
  SS_LAUNCH_CHECK();
  if (!a.x_in_a) {
    k_pass<PASS_X><<<gs, PT, K->smem_pass, st>>>(a);
    SS_LAUNCH_CHECK();
  }
  return SS_OK;
}

static int tick_dim(const ss_krylov* K) { return K->a.kind == 0 ? K->a.op.dim : 2; }

// Device-side loop control: after every body of ticks, keep looping while some mode is not done
// and the tick cap is not reached (the whole solve is ONE graph launch, no host round trips).
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* __restrict__ n_done, int nb,
                            long long* loop, int per_body) {
  const long long t = (loop[0] += per_body);
  cudaGraphSetConditional(h, (*n_done < nb && t < loop[1]) ? 1u : 0u);
}

static int get_while_graph(ss_krylov* K, int nb, int jacobi, cudaGraphExec_t* out) {
  const int64_t key = (int64_t)nb * 4 + jacobi * 2 + 1;
  auto it = K->graphs.find(key);
  if (it != K->graphs.end()) { *out = it->second; return SS_OK; }
  KArgs a = K->a;
  a.nb = nb;
  a.jacobi = jacobi;
  cudaGraph_t g;
  SS_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  SS_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  SS_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  SS_CUDA(cudaStreamBeginCaptureToGraph(K->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int rc = SS_OK;
  for (int t = 0; t < K->ticks_per_graph && !rc; ++t)
    rc = tick_dim(K) == 3 ? launch_tick<3>(K, a, K->cap_stream) : launch_tick<2>(K, a, K->cap_stream);
  if (!rc) {
    k_loop_cond<<<1, 1, 0, K->cap_stream>>>(h, a.n_done, nb, a.loop, K->ticks_per_graph);
    if (cudaGetLastError() != cudaSuccess) rc = SS_ERR_CUDA;
  }
  cudaError_t e = cudaStreamEndCapture(K->cap_stream, &body);
  if (rc || e != cudaSuccess) {
    cudaGraphDestroy(g);
    ss_set_error(std::string("conditional graph capture failed: ") + cudaGetErrorString(e));
    return rc ? rc : SS_ERR_CUDA;
  }
  cudaGraphExec_t ex;
  SS_CUDA(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  K->graphs[key] = ex;
  *out = ex;
  return SS_OK;
}

static int get_graph(ss_krylov* K, int nb, int jacobi, cudaGraphExec_t* out) {
  const int64_t key = (int64_t)nb * 4 + jacobi * 2;
  auto it = K->graphs.find(key);
  if (it != K->graphs.end()) { *out = it->second; return SS_OK; }
  KArgs a = K->a;
  a.nb = nb;
  a.jacobi = jacobi;
  cudaGraph_t g;
  SS_CUDA(cudaStreamBeginCapture(K->cap_stream, cudaStreamCaptureModeThreadLocal));
  int rc = SS_OK;
  for (int t = 0; t < K->ticks_per_graph && !rc; ++t)
    rc = tick_dim(K) == 3 ? launch_tick<3>(K, a, K->cap_stream) : launch_tick<2>(K, a, K->cap_stream);
  cudaError_t e = cudaStreamEndCapture(K->cap_stream, &g);
  if (rc) return rc;
  if (e != cudaSuccess) { ss_set_error(std::string("graph capture failed: ") + cudaGetErrorString(e)); return SS_ERR_CUDA; }
  cudaGraphExec_t ex;
  SS_CUDA(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  K->graphs[key] = ex;
  *out = ex;
  return SS_OK;
}

// Persistent fused tick: shared-memory budget and grid (one CTA per SM) on first use.  The ring
// shrinks to what the static shared state leaves of the 227 KB per CTA (chunking does not change
// any sum).  Returns false when the fused kernel cannot run this workspace.
template <int DIM>
static bool fused_setup(ss_krylov* K) {
  if (K->fused_grid != 0) return K->fused_grid > 0;
  K->fused_grid = -1;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, (const void*)k_tick_fused<DIM>) != cudaSuccess) { cudaGetLastError(); return false; }
  const int dyn_max = 227 * 1024 - (int)fa.sharedSizeBytes;
  // the ring must equal the four-kernel tick's (pass C/X chunking sets their slice sums)
  const int elems = K->a.smem_elems;
  if (elems > dyn_max / (int)sizeof(double2)) return false;
  if (cudaFuncSetAttribute((const void*)k_tick_fused<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           elems * (int)sizeof(double2)) != cudaSuccess) { cudaGetLastError(); return false; }
  int dev = 0, sms = 0, coop = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop || cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tick_fused<DIM>, PT,
                                                            (size_t)elems * sizeof(double2)) != cudaSuccess ||
      per_sm < 1) { cudaGetLastError(); return false; }
  K->fused_elems = elems;
  K->fused_grid = sms;
  return true;
}

static bool fused_usable(ss_krylov* K) {
  if (!K->fused || (K->a.kind == 0 && K->a.row_spmv)) return false;
  return tick_dim(K) == 3 ? fused_setup<3>(K) : fused_setup<2>(K);
}

static int launch_fused(ss_krylov* K, const KArgs& a0, int nticks, int tick0, cudaStream_t st) {
  KArgs a = a0;
  a.fused = 1;
  a.x_in_a = 1;
  a.smem_elems = K->fused_elems;
  a.ptime = K->ptime;
  void* args[] = {(void*)&a, (void*)&nticks, (void*)&tick0};
  const void* f = tick_dim(K) == 3 ? (const void*)k_tick_fused<3> : (const void*)k_tick_fused<2>;
  SS_CUDA(cudaLaunchCooperativeKernel(f, dim3(K->fused_grid), dim3(PT), args,
                                      (size_t)K->fused_elems * sizeof(double2), st));
  return SS_OK;
}

// Solve nb modes.  rhs/x0 are read from the engine's own RHS/X buffers (see ss_krylov_buffers)
// when rhs_dev / x_dev are null, otherwise copied in (device pointers, leading dimension ld_in).
// On return X holds the solutions (also copied to x_dev when given).
// out_int[b*6 + {0: iterations, 1: converged flag, 2: breakdown, 3: phase, 4: history length, 5: zero rhs}]
// out_dbl[b*4 + {0: true residual at last cycle end, 1: last estimate, 2: ||b||, 3: target}]
extern "C" int ss_krylov_solve(ss_krylov* K, int nb, const double* omegas_host, const int* sets_host,
                               const double* rhs_dev, double* x_dev, int64_t ld_in, int use_x0, double tol,
                               int64_t maxiter, int jacobi, void* stream_, int64_t* out_int, double* out_dbl) {
  if (!K || nb < 1 || nb > K->max_batch || !omegas_host) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (!(tol > 0.0 && tol < 1.0)) { ss_set_error("tolerance must lie in (0, 1)"); return SS_ERR_ARG; }
  if (maxiter < 0 || maxiter > INT32_MAX) { ss_set_error("bad maxiter"); return SS_ERR_ARG; }
  SS_CUDA(cudaSetDevice(K->device));
  cudaStream_t st = (cudaStream_t)stream_;
  KArgs a = K->a;
  a.nb = nb;
  a.jacobi = jacobi;
  const int64_t launches0 = ss_launch_counter();
  std::vector<ModeCtl> ctl(nb);
  for (int b = 0; b < nb; ++b) {
    ModeCtl c{};
    c.phase = PH_IDLE;
    c.maxiter = (int)maxiter;
    c.restart = a.restart;
    c.tol = tol;
    c.omega = omegas_host[b];
    c.set = sets_host ? sets_host[b] : b;
    ctl[b] = c;
  }
  SS_CUDA(cudaMemcpyAsync(a.ctl, ctl.data(), sizeof(ModeCtl) * nb, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemsetAsync(a.n_done, 0, sizeof(int), st));
  SS_CUDA(cudaMemsetAsync(a.loop + 2, 0, sizeof(long long), st));
  // election / block-dealing counters start from zero (every kernel also leaves them zeroed)
  SS_CUDA(cudaMemsetAsync(a.counters, 0, sizeof(int) * 8 * (size_t)K->max_batch, st));
  if (rhs_dev)
    SS_CUDA(cudaMemcpy2DAsync(a.RHS, a.ld * sizeof(double2), rhs_dev, ld_in * sizeof(double2), a.n * sizeof(double2),
                              nb, cudaMemcpyDeviceToDevice, st));
  if (use_x0 && x_dev)
    SS_CUDA(cudaMemcpy2DAsync(a.X, a.ld * sizeof(double2), x_dev, ld_in * sizeof(double2), a.n * sizeof(double2), nb,
                              cudaMemcpyDeviceToDevice, st));
  else if (!use_x0)
    SS_CUDA(cudaMemsetAsync(a.X, 0, sizeof(double2) * a.ld * nb, st));
  if (tick_dim(K) == 3) k_init<3><<<nb * a.nseg, PT, 0, st>>>(a);
  else k_init<2><<<nb * a.nseg, PT, 0, st>>>(a);
  SS_LAUNCH_CHECK();
  // tick bound: every mode finishes within maxiter inner ticks + 2 ticks per cycle
  const int64_t max_ticks = maxiter + 3 * (maxiter / std::max<int64_t>(1, std::min<int64_t>(a.restart, maxiter + 1)) + 2) + 16;
  int64_t ticks = 0;
  cudaGraphExec_t g = nullptr;
  int rc = SS_OK;
  const bool fused = fused_usable(K);
  if (K->device_loop && !fused) {
    rc = get_while_graph(K, nb, jacobi, &g);
    if (rc) K->device_loop = 0;   // fall back to the host-polled loop
  }
  if (K->device_loop && !fused) {
    long long lp[2] = {0, (long long)max_ticks + 2 * K->ticks_per_graph};
    SS_CUDA(cudaMemcpyAsync(a.loop, lp, sizeof(lp), cudaMemcpyHostToDevice, st));
    SS_CUDA(cudaGraphLaunch(g, st));
    SS_CUDA(cudaMemcpyAsync(lp, a.loop, sizeof(lp), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaStreamSynchronize(st));
    ticks = lp[0];
    ss_count_launch((ticks / K->ticks_per_graph) * ((a.x_in_a ? 4 : 5) * K->ticks_per_graph + 1));
    int done = 0;
    SS_CUDA(cudaMemcpy(&done, a.n_done, sizeof(int), cudaMemcpyDeviceToHost));
    if (done < nb) {
      ss_set_error("GMRES tick bound exceeded (internal state machine error)");
      return SS_ERR_STATE;
    }
  }
  rc = (K->device_loop && !fused) || fused ? SS_OK : get_graph(K, nb, jacobi, &g);
  if (rc) return rc;
  const int per_graph_launches = fused ? 1 : (a.x_in_a ? 4 : 5) * K->ticks_per_graph;
  int it = 0;
  bool finished = K->device_loop != 0 && !fused;
  while (!finished) {
    if (fused) {
      if ((rc = launch_fused(K, a, K->ticks_per_graph, (int)ticks, st))) return rc;
    } else {
      SS_CUDA(cudaGraphLaunch(g, st));
    }
    ss_count_launch(per_graph_launches);
    ticks += K->ticks_per_graph;
    SS_CUDA(cudaMemcpyAsync(K->h_done + (it & 1), a.n_done, sizeof(int), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaEventRecord(K->ev[it & 1], st));
    if (it > 0) {
      SS_CUDA(cudaEventSynchronize(K->ev[(it - 1) & 1]));
      if (K->h_done[(it - 1) & 1] >= nb) finished = true;
    }
    if (ticks > max_ticks + 4 * K->ticks_per_graph) {
      ss_set_error("GMRES tick bound exceeded (internal state machine error)");
      return SS_ERR_STATE;
    }
    ++it;
  }
  if (it > 0) SS_CUDA(cudaEventSynchronize(K->ev[(it - 1) & 1]));
  k_finalize<<<dim3(64, nb), 256, 0, st>>>(a);
  SS_LAUNCH_CHECK();
  if (x_dev)
    SS_CUDA(cudaMemcpy2DAsync(x_dev, ld_in * sizeof(double2), a.X, a.ld * sizeof(double2), a.n * sizeof(double2), nb,
                              cudaMemcpyDeviceToDevice, st));
  SS_CUDA(cudaMemcpyAsync(ctl.data(), a.ctl, sizeof(ModeCtl) * nb, cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  K->last_ticks = ticks;
  K->last_launches = ss_launch_counter() - launches0;
  if (fused && K->ptime) {   // per-tick phase durations (us): spmv, A, B, C
    const int64_t nt = std::min<int64_t>(ticks, FUSED_PROF_TICKS);
    std::vector<long long> h((size_t)nt * 5);
    SS_CUDA(cudaMemcpy(h.data(), K->ptime, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(getenv("SS_FUSED_PROF"), "w")) {
      for (int64_t t = 0; t < nt; ++t) {
        const long long* r = h.data() + t * 5;
        if (r[4] <= r[0]) break;
        fprintf(f, "%.3f,%.3f,%.3f,%.3f\n", 1e-3 * (r[1] - r[0]), 1e-3 * (r[2] - r[1]), 1e-3 * (r[3] - r[2]),
                1e-3 * (r[4] - r[3]));
      }
      fclose(f);
    }
  }
  for (int b = 0; b < nb; ++b) {
    if (out_int) {
      out_int[b * 6 + 0] = ctl[b].iters;
      out_int[b * 6 + 1] = ctl[b].converged;
      out_int[b * 6 + 2] = ctl[b].breakdown;
      out_int[b * 6 + 3] = ctl[b].phase;
      out_int[b * 6 + 4] = ctl[b].hist_len;
      out_int[b * 6 + 5] = ctl[b].zero_x;
    }
    if (out_dbl) {
      out_dbl[b * 4 + 0] = ctl[b].true_res;
      out_dbl[b * 4 + 1] = ctl[b].est;
      out_dbl[b * 4 + 2] = ctl[b].bnorm;
      out_dbl[b * 4 + 3] = ctl[b].target;
    }
  }
  return SS_OK;
}

// Tick at which each of the last solve's nb modes finished (0 = before the first tick).
extern "C" int ss_krylov_done_ticks(const ss_krylov* K, int nb, int64_t* out_host) {
  if (!K || !out_host || nb < 1 || nb > K->max_batch) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  std::vector<ModeCtl> ctl(nb);
  SS_CUDA(cudaSetDevice(K->device));
  SS_CUDA(cudaMemcpy(ctl.data(), K->a.ctl, sizeof(ModeCtl) * nb, cudaMemcpyDeviceToHost));
  for (int b = 0; b < nb; ++b) out_host[b] = ctl[b].done_tick;
  return SS_OK;
}

extern "C" int ss_krylov_last_stats(const ss_krylov* K, int64_t* ticks, int64_t* launches) {
  if (!K) { ss_set_error("null argument"); return SS_ERR_ARG; }
  if (ticks) *ticks = K->last_ticks;
  if (launches) *launches = K->last_launches;
  return SS_OK;
}

extern "C" int ss_krylov_history(const ss_krylov* K, int mode, int64_t count, double* out) {
  if (!K || !out || mode < 0 || mode >= K->max_batch) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  count = std::min(count, K->a.hist_cap);
  if (count > 0)
    SS_CUDA(cudaMemcpy(out, K->a.hist + (size_t)mode * K->a.hist_cap, sizeof(double) * count, cudaMemcpyDeviceToHost));
  return SS_OK;
}

// One isolated basis pass (bench / profiling): runs k_pass<which> (A, B or C) for nb modes, all
// forced into phase INNER at basis index k (J = k+1 vectors).  Returns algorithmic bytes in *bytes.
__global__ void k_force_inner(KArgs a, int k) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nb) return;
  a.ctl[b].phase = PH_INNER;
  a.ctl[b].k = k;
  a.ctl[b].maxiter = 0x7fffffff;
  a.ctl[b].iters = 0;
  a.ctl[b].target = -1.0;
  a.ctl[b].beta = 1.0;
  for (int j = 0; j <= k; ++j) a.qs[b * a.jcap + j] = 1.0;
}

// Bench input: w = 1 on the active rows (so ||w|| > 0 in pass C), zero projection coefficients.
__global__ void k_bench_fill(KArgs a) {
  const int64_t total = (int64_t)a.nb * a.ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i % a.ld;
    a.W[i] = make_double2(row < a.n ? 1.0 : 0.0, 0.0);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)a.nb * a.jcap;
       i += (int64_t)gridDim.x * blockDim.x) {
    a.C1[i] = make_double2(0.0, 0.0);
    a.C2[i] = make_double2(0.0, 0.0);
  }
}

extern "C" int ss_krylov_bench_pass(ss_krylov* K, int nb, int k, int which, int reps, void* stream_, float* ms,
                                    int64_t* bytes) {
  if (!K || nb < 1 || nb > K->max_batch || k < 0 || k >= K->a.restart) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  KArgs a = K->a;
  a.nb = nb;
  k_force_inner<<<(nb + 127) / 128, 128, 0, st>>>(a, k);
  SS_LAUNCH_CHECK();
  cudaEvent_t e0, e1;
  SS_CUDA(cudaEventCreate(&e0));
  SS_CUDA(cudaEventCreate(&e1));
  const unsigned gs = (unsigned)(nb * a.nseg);
  k_bench_fill<<<4 * 148, 256, 0, st>>>(a);
  SS_LAUNCH_CHECK();
  auto one = [&]() {
    if (which == PASS_A) k_pass<PASS_A><<<gs, PT, K->smem_pass, st>>>(a);
    else if (which == PASS_B) k_pass<PASS_B><<<gs, PT, K->smem_pass, st>>>(a);
    else k_pass<PASS_C><<<gs, PT, K->smem_pass, st>>>(a);
  };
  // warm-up
  one();
  SS_LAUNCH_CHECK();
  if (which == PASS_C) k_force_inner<<<(nb + 127) / 128, 128, 0, st>>>(a, k);
  SS_CUDA(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r) {
    one();
    SS_LAUNCH_CHECK();
    // pass C advances k (Givens step): re-arm (a ~2 us kernel, included in the time)
    if (which == PASS_C) k_force_inner<<<(nb + 127) / 128, 128, 0, st>>>(a, k);
  }
  SS_CUDA(cudaEventRecord(e1, st));
  SS_CUDA(cudaEventSynchronize(e1));
  SS_CUDA(cudaEventElapsedTime(ms, e0, e1));
  *ms /= reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const int64_t J = k + 1;
  // A: read Q (J vectors) + w;  B: read Q + w, write w;  C: read Q + w, write q_{k+1}
  *bytes = (int64_t)nb * 16 * a.n * (J + (which == PASS_A ? 1 : 2));
  return SS_OK;
}

// True relative residuals ||b - A x|| / ||b|| (||A x|| when b = 0) of the workspace's X for nb modes.
extern "C" int ss_krylov_residuals(ss_krylov* K, int nb, void* stream_, double* out_host) {
  if (!K || nb < 1 || nb > K->max_batch || !out_host) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  KArgs a = K->a;
  a.nb = nb;
  if (K->a.kind == 0 && K->a.op.dim == 3) k_true_resid<3><<<nb * a.nsb, PT, 0, st>>>(a);
  else k_true_resid<2><<<nb * a.nsb, PT, 0, st>>>(a);
  SS_LAUNCH_CHECK();
  std::vector<double2> h((size_t)nb * a.nsb);
  SS_CUDA(cudaMemcpyAsync(h.data(), a.spart, sizeof(double2) * h.size(), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < nb; ++b) {
    double tt = 0, bb = 0;
    for (int q = 0; q < a.nsb; ++q) { tt += h[(size_t)b * a.nsb + q].x; bb += h[(size_t)b * a.nsb + q].y; }
    out_host[b] = bb == 0.0 ? std::sqrt(tt) : std::sqrt(tt) / std::sqrt(bb);
  }
  return SS_OK;
}

// Copy nb rows between caller device buffers and the workspace (dir 0: caller -> RHS, 1: caller -> X,
// 2: X -> caller).
extern "C" int ss_krylov_copy(ss_krylov* K, int nb, int dir, double* buf_dev, int64_t ld_in, void* stream_) {
  if (!K || nb < 1 || nb > K->max_batch || !buf_dev) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream_;
  const KArgs& a = K->a;
  const size_t w = (size_t)a.n * sizeof(double2);
  if (dir == 0)
    SS_CUDA(cudaMemcpy2DAsync(a.RHS, a.ld * 16, buf_dev, ld_in * 16, w, nb, cudaMemcpyDeviceToDevice, st));
  else if (dir == 1)
    SS_CUDA(cudaMemcpy2DAsync(a.X, a.ld * 16, buf_dev, ld_in * 16, w, nb, cudaMemcpyDeviceToDevice, st));
  else
    SS_CUDA(cudaMemcpy2DAsync(buf_dev, ld_in * 16, a.X, a.ld * 16, w, nb, cudaMemcpyDeviceToDevice, st));
  return SS_OK;
}

// Jacobi scale of the CSR operator's value set `set` (jacobi_precondition on a matrix).
extern "C" int ss_krylov_csr_scale(const ss_krylov* K, int set, double* out_host) {
  if (!K || K->a.kind != 1 || !K->a.csr.scale || !out_host) { ss_set_error("no CSR scale"); return SS_ERR_ARG; }
  SS_CUDA(cudaMemcpy(out_host, K->a.csr.scale + (size_t)set * K->a.csr.n, sizeof(double2) * K->a.csr.n,
                     cudaMemcpyDeviceToHost));
  return SS_OK;
}

// Instrumented solve for the roofline: identical kernels launched one by one (no graph) with
// CUDA events on the launching stream between them; accumulates per-kernel-kind device time and
// the algorithmic bytes each kind moved.  kind: 0 spmv, 1 passA, 2 passB, 3 passC, 4 passX.
// ms_out[5], bytes_out[5], launches_out[5].
template <int DIM>
static int profile_ticks(ss_krylov* K, const KArgs& a, cudaStream_t st, int64_t max_ticks, double* ms_out,
                         int64_t* launches_out) {
  const unsigned gs = (unsigned)(a.nb * a.nseg);
  cudaEvent_t ev[6];
  for (auto& e : ev) SS_CUDA(cudaEventCreate(&e));
  int64_t tick = 0;
  int done = 0;
  unsigned sgrid;
  size_t ssmem;
  tick_spmv_launch_dims<DIM>(K, a, &sgrid, &ssmem);
  while (tick < max_ticks) {
    SS_CUDA(cudaEventRecord(ev[0], st));
    if (ssmem) k_tick_spmv_stream<DIM><<<sgrid, PT, ssmem, st>>>(a);
    else if (a.kind == 0 && a.row_spmv) k_tick_spmv<DIM, 1><<<sgrid, PT, 0, st>>>(a);
    else k_tick_spmv<DIM, 0><<<sgrid, PT, 0, st>>>(a);
    SS_LAUNCH_CHECK();
    SS_CUDA(cudaEventRecord(ev[1], st));
    k_pass<PASS_A><<<gs, PT, K->smem_pass, st>>>(a);
    SS_LAUNCH_CHECK();
    SS_CUDA(cudaEventRecord(ev[2], st));
    k_pass<PASS_B><<<gs, PT, K->smem_pass, st>>>(a);
    SS_LAUNCH_CHECK();
    SS_CUDA(cudaEventRecord(ev[3], st));
    k_pass<PASS_C><<<gs, PT, K->smem_pass, st>>>(a);
    SS_LAUNCH_CHECK();
    SS_CUDA(cudaEventRecord(ev[4], st));
    if (!a.x_in_a) {
      k_pass<PASS_X><<<gs, PT, K->smem_pass, st>>>(a);
      SS_LAUNCH_CHECK();
    }
    SS_CUDA(cudaEventRecord(ev[5], st));
    SS_CUDA(cudaMemcpyAsync(K->h_done, a.n_done, sizeof(int), cudaMemcpyDeviceToHost, st));
    SS_CUDA(cudaEventSynchronize(ev[5]));
    static FILE* dump = getenv("SS_PROFILE_DUMP") ? fopen(getenv("SS_PROFILE_DUMP"), "w") : nullptr;
    for (int q = 0; q < 5; ++q) {
      float ms = 0;
      SS_CUDA(cudaEventElapsedTime(&ms, ev[q], ev[q + 1]));
      ms_out[q] += ms;
      launches_out[q] += 1;
      if (dump) fprintf(dump, q < 4 ? "%.4f," : "%.4f\n", ms);
    }
    if (dump) fflush(dump);
    ++tick;
    done = K->h_done[0];
    if (done >= a.nb) break;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return SS_OK;
}

extern "C" int ss_krylov_profile(ss_krylov* K, int nb, const double* omegas_host, double tol, int64_t maxiter,
                                 int jacobi, void* stream_, double* ms_out, int64_t* bytes_out, int64_t* launches_out) {
  if (!K || nb < 1 || nb > K->max_batch || !omegas_host || !ms_out || !bytes_out || !launches_out) {
    ss_set_error("bad arguments");
    return SS_ERR_ARG;
  }
  SS_CUDA(cudaSetDevice(K->device));
  cudaStream_t st = (cudaStream_t)stream_;
  KArgs a = K->a;
  a.nb = nb;
  a.jacobi = jacobi;
  std::vector<ModeCtl> ctl(nb);
  for (int b = 0; b < nb; ++b) {
    ModeCtl c{};
    c.maxiter = (int)maxiter;
    c.restart = a.restart;
    c.tol = tol;
    c.omega = omegas_host[b];
    c.set = b;
    ctl[b] = c;
  }
  SS_CUDA(cudaMemcpyAsync(a.ctl, ctl.data(), sizeof(ModeCtl) * nb, cudaMemcpyHostToDevice, st));
  SS_CUDA(cudaMemsetAsync(a.n_done, 0, sizeof(int), st));
  SS_CUDA(cudaMemsetAsync(a.loop + 2, 0, sizeof(long long), st));
  // election / block-dealing counters start from zero (every kernel also leaves them zeroed)
  SS_CUDA(cudaMemsetAsync(a.counters, 0, sizeof(int) * 8 * (size_t)K->max_batch, st));
  SS_CUDA(cudaMemsetAsync(a.X, 0, sizeof(double2) * a.ld * nb, st));
  SS_CUDA(cudaMemsetAsync(a.bytes, 0, sizeof(unsigned long long) * 8, st));
  if (tick_dim(K) == 3) k_init<3><<<nb * a.nseg, PT, 0, st>>>(a);
  else k_init<2><<<nb * a.nseg, PT, 0, st>>>(a);
  SS_LAUNCH_CHECK();
  for (int q = 0; q < 5; ++q) { ms_out[q] = 0; launches_out[q] = 0; }
  const int64_t max_ticks = maxiter + 3 * (maxiter / std::max<int64_t>(1, std::min<int64_t>(a.restart, maxiter + 1)) + 2) + 16;
  int rc = tick_dim(K) == 3 ? profile_ticks<3>(K, a, st, max_ticks, ms_out, launches_out)
                            : profile_ticks<2>(K, a, st, max_ticks, ms_out, launches_out);
  if (rc) return rc;
  unsigned long long hb[8];
  SS_CUDA(cudaMemcpyAsync(hb, a.bytes, sizeof(hb), cudaMemcpyDeviceToHost, st));
  SS_CUDA(cudaStreamSynchronize(st));
  for (int q = 0; q < 5; ++q) bytes_out[q] = (int64_t)hb[q];
  return SS_OK;
}
