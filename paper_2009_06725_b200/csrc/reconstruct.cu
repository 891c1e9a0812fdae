// Fused inverse-Fourier reconstruction of all requested time samples in one launch.
//
// Restates reconstruct (reference pkg/src/spectralstokes/spectral.py:308-317):
//   out[t][i] = sum_b Re(field_b[i] * phase_b(t)),  accumulated in mode-list order from +0.0,
// with phase_b(t) = exp(1j*omega_b*t) computed by the caller exactly as the reference does.
// Products use explicit round-to-nearest intrinsics (no FMA contraction) so the sum reproduces
// numpy's `u += np.real(v * phase)` operation by operation.
// Traffic: each modal value is read once (16 B x nb x n) and every sample written once (8 B x nt x n).
#include "ss_common.h"

template <int MAXB>
__global__ void __launch_bounds__(256) k_reconstruct(int nb, int nt, int64_t n, const double2* __restrict__ fields,
                                                     const double2* __restrict__ phases, double* __restrict__ out) {
  extern __shared__ double2 ph[];   // [nb][nt]
  for (int q = threadIdx.x; q < nb * nt; q += blockDim.x) ph[q] = phases[q];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v[MAXB];
#pragma unroll
    for (int b = 0; b < MAXB; ++b) v[b] = b < nb ? fields[(size_t)b * n + i] : make_double2(0.0, 0.0);
    for (int t = 0; t < nt; ++t) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        if (b < nb) {
          const double2 p = ph[b * nt + t];
          acc = __dadd_rn(acc, __dsub_rn(__dmul_rn(v[b].x, p.x), __dmul_rn(v[b].y, p.y)));
        }
      }
      out[(size_t)t * n + i] = acc;
    }
  }
}

// Generic path for large mode counts: modes streamed from L1/L2 per sample.
__global__ void __launch_bounds__(256) k_reconstruct_many(int nb, int nt, int64_t n, const double2* __restrict__ fields,
                                                          const double2* __restrict__ phases, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    for (int t = 0; t < nt; ++t) {
      double acc = 0.0;
      for (int b = 0; b < nb; ++b) {
        const double2 v = fields[(size_t)b * n + i];
        const double2 p = phases[(size_t)b * nt + t];
        acc = __dadd_rn(acc, __dsub_rn(__dmul_rn(v.x, p.x), __dmul_rn(v.y, p.y)));
      }
      out[(size_t)t * n + i] = acc;
    }
  }
}

extern "C" int ss_reconstruct(int nb, int nt, int64_t n, const double* fields_dev, const double* phases_dev,
                              double* out_dev, void* stream_) {
  if (nb < 1 || nt < 1 || n < 0 || !fields_dev || !phases_dev || !out_dev) { ss_set_error("bad arguments"); return SS_ERR_ARG; }
  if (n == 0) return SS_OK;
  cudaStream_t st = (cudaStream_t)stream_;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
  const size_t smem = sizeof(double2) * nb * nt;
  const double2* f = (const double2*)fields_dev;
  const double2* p = (const double2*)phases_dev;
  if (nb <= 16 && smem <= 48 * 1024) {
    k_reconstruct<16><<<(unsigned)blocks, 256, smem, st>>>(nb, nt, n, f, p, out_dev);
  } else if (nb <= 32 && smem <= 48 * 1024) {
    k_reconstruct<32><<<(unsigned)blocks, 256, smem, st>>>(nb, nt, n, f, p, out_dev);
  } else {
    k_reconstruct_many<<<(unsigned)blocks, 256, 0, st>>>(nb, nt, n, f, p, out_dev);
  }
  SS_LAUNCH_CHECK();
  return SS_OK;
}
