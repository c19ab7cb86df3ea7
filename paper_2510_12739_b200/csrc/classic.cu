// classic.cu — the classical baseline receiver on the GPU: per-RE LMMSE
// combining over the receive antennas and max-log demapping (classic.cpp missing from
// the snapshot), fed either by the LS + interpolation channel estimate the featurizer already computes
// (ls_lmmse) or by the true channel (perfect_csi_lmmse).
//
//   x_hat = h^H y / (h^H h + s2)                           (unit-energy symbols, interference as noise)
//   unbiased z = x_hat / mu = h^H y / h^H h,  mu = h^H h / (h^H h + s2),  noise var nu = s2 / h^H h
//   LLR_b = (min_{s: b=0} |z - s|^2 - min_{s: b=1} |z - s|^2) / nu     (positive => bit 1)
//
// Gray QAM is separable (qam.cpp:23-52: even bits -> I, odd bits -> Q), so every minimum is a 1-D search
// over the sqrt(M) levels of one axis — exact max-log, equal to the exhaustive 2-D search.
// An all-zero channel gives z = 0 with infinite noise variance: LLRs are 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "common.h"
#include "kernels.h"

namespace cnrx {

namespace {

// unnormalised level of an axis from its bits (qam.cpp:23-30); nb_axis = bits per axis
__device__ __forceinline__ float level(int v, int nb_axis) {
  const float s0 = 1.f - 2.f * static_cast<float>(v & 1);
  if (nb_axis == 1) return s0;
  const float s1 = 1.f - 2.f * static_cast<float>((v >> 1) & 1);
  if (nb_axis == 2) return s0 * (2.f - s1);
  const float s2 = 1.f - 2.f * static_cast<float>((v >> 2) & 1);
  return s0 * (4.f - s1 * (2.f - s2));
}

// feat: [B,T,F,6N] (Re y, Im y, Re x_p, Im x_p, Re h_ls, Im h_ls per antenna) or null with y/h given
__global__ void lmmse_demap_kernel(const float* __restrict__ feat, const float2* __restrict__ y,
                                   const float2* __restrict__ h, const float* __restrict__ noise_var, int64_t B,
                                   int T, int F, int N, int nb, float* __restrict__ llr) {
  const int64_t total = B * T * F;
  const int nba = nb / 2;
  const float nf = nb == 2 ? 0.70710678118654752f : nb == 4 ? 0.31622776601683794f : 0.15430334996209191f;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / (static_cast<int64_t>(T) * F);
    float g = 0.f, nr = 0.f, ni = 0.f;
    for (int a = 0; a < N; ++a) {
      float yr, yi, hr, hi;
      if (feat) {
        const float* fp = feat + i * 6 * N + 6 * a;
        yr = fp[0];
        yi = fp[1];
        hr = fp[4];
        hi = fp[5];
      } else {
        const float2 yy = y[i * N + a], hh = h[i * N + a];
        yr = yy.x;
        yi = yy.y;
        hr = hh.x;
        hi = hh.y;
      }
      g += hr * hr + hi * hi;
      nr += hr * yr + hi * yi;  // conj(h) * y
      ni += hr * yi - hi * yr;
    }
    float* out = llr + i * nb;
    if (!(g > 0.f)) {
      for (int k = 0; k < nb; ++k) out[k] = 0.f;
      continue;
    }
    const float zr = nr / g, zi = ni / g;
    const float inv_nu = g / noise_var[b];
    for (int k = 0; k < nb; ++k) {
      const float zc = (k & 1) ? zi : zr;  // even bits -> I axis, odd -> Q axis
      const int bit_in_axis = k >> 1;
      float d0 = 3.4e38f, d1 = 3.4e38f;
      for (int v = 0; v < (1 << nba); ++v) {
        const float e = zc - level(v, nba) * nf;
        const float d = e * e;
        if ((v >> bit_in_axis) & 1) d1 = fminf(d1, d);
        else d0 = fminf(d0, d);
      }
      out[k] = (d0 - d1) * inv_nu;
    }
  }
}

}  // namespace

const char* launch_lmmse_demap(const float* feat, const float2* y, const float2* h, const float* noise_var, int64_t B,
                               int T, int F, int N, int bits, float* llr, cudaStream_t s) {
  const int64_t total = B * T * F;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  lmmse_demap_kernel<<<blocks, 256, 0, s>>>(feat, y, h, noise_var, B, T, F, N, bits, llr);
  CNRX_CUDA(cudaGetLastError());
  return "lmmse_demap_kernel";
}

}  // namespace cnrx
