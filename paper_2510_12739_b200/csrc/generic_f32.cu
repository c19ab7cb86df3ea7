// generic_f32.cu — fp32 CUDA-core kernels for CNRX_FP32 plans, in the reference layout [B,T,F,C].
//
// The fp32 path is the one BASELINE config 1 names ("CoNet-small, fp32") and the fp32 leg of the
// config-5 sweep.  It is BIT-EXACT with the reference: every kernel performs the reference's float
// operations in the reference's order with the reference's rounding — conv accumulates bias, then
// taps (dt, df) and input channels in order with separately rounded multiply and add
// (yrow[co] += xv * wrow[co], kernels.hpp:78-82; x86-64 has no FMA contraction), eval BN applies the
// host-folded float scale/shift (norms.hpp:81-95), layer norm runs in double (norms.hpp:155-191).
// Each LayerOp has a kernel (network.hpp:380-420); the plan compiler fuses a conv with the
// single-consumer BN / ReLU / add|mul chain that follows it without changing any rounding.
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.h"

namespace cnrx {

namespace {

constexpr int kCot = 16;  // output channels per block of the direct conv

// Direct "same" conv, stride 1 (kernels.hpp:47-91): one thread = one output pixel x 16 channels.
__global__ void __launch_bounds__(128) conv_f32_kernel(const ConvF32 p) {
  extern __shared__ float sw[];  // [kh*kw][cin][kCot]
  const int co0 = blockIdx.y * kCot;
  const int ncot = min(kCot, p.cout - co0);
  const int taps = p.kh * p.kw;
  for (int i = threadIdx.x; i < taps * p.cin * kCot; i += blockDim.x) {
    const int co = i % kCot;
    const int tci = i / kCot;  // tap*cin + ci
    sw[i] = co < ncot ? p.w[static_cast<int64_t>(tci) * p.cout + co0 + co] : 0.f;
  }
  __syncthreads();
  const int64_t pix = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t npix = static_cast<int64_t>(p.B) * p.T * p.F;
  if (pix >= npix) return;
  const int f = static_cast<int>(pix % p.F);
  const int t = static_cast<int>((pix / p.F) % p.T);
  const int64_t b = pix / (static_cast<int64_t>(p.F) * p.T);
  float acc[kCot];
#pragma unroll
  for (int c = 0; c < kCot; ++c) acc[c] = (p.bias && c < ncot) ? p.bias[co0 + c] : 0.f;
  const int oh = p.kh / 2, ow = p.kw / 2;
  for (int dt = 0; dt < p.kh; ++dt) {
    const int ti = t + dt - oh;
    if (ti < 0 || ti >= p.T) continue;
    for (int df = 0; df < p.kw; ++df) {
      const int fi = f + (df - ow) * p.dil_f;
      if (fi < 0 || fi >= p.F) continue;
      const float* xr = p.x + ((b * p.T + ti) * p.F + fi) * p.cin;
      const float* wt = sw + (dt * p.kw + df) * p.cin * kCot;
      int ci = 0;
      if ((p.cin & 3) == 0) {
        for (; ci < p.cin; ci += 4) {
          const float4 xv = *reinterpret_cast<const float4*>(xr + ci);
          const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4* w4 = reinterpret_cast<const float4*>(wt + (ci + u) * kCot);
#pragma unroll
            for (int q = 0; q < kCot / 4; ++q) {
              const float4 wv = w4[q];
              acc[4 * q + 0] = __fadd_rn(acc[4 * q + 0], __fmul_rn(xs[u], wv.x));
              acc[4 * q + 1] = __fadd_rn(acc[4 * q + 1], __fmul_rn(xs[u], wv.y));
              acc[4 * q + 2] = __fadd_rn(acc[4 * q + 2], __fmul_rn(xs[u], wv.z));
              acc[4 * q + 3] = __fadd_rn(acc[4 * q + 3], __fmul_rn(xs[u], wv.w));
            }
          }
        }
      }
      for (; ci < p.cin; ++ci) {
        const float xv = xr[ci];
#pragma unroll
        for (int c = 0; c < kCot; ++c) acc[c] = __fadd_rn(acc[c], __fmul_rn(xv, wt[ci * kCot + c]));
      }
    }
  }
  float* yr = p.y + pix * p.cout + co0;
  const float* orow = p.other ? p.other + pix * p.cout + co0 : nullptr;
#pragma unroll
  for (int c = 0; c < kCot; ++c) {
    if (c >= ncot) break;
    float v = acc[c];
    if (p.aff_s) v = __fadd_rn(__fmul_rn(v, p.aff_s[co0 + c]), p.aff_t[co0 + c]);
    if (p.relu) v = v > 0.f ? v : 0.f;
    if (p.other_op == 6) v = __fadd_rn(v, orow[c]);
    if (p.other_op == 7) v = __fmul_rn(v, orow[c]);
    yr[c] = v;
  }
}

// Packed fp32 pairs, each lane rounded separately (inline PTX: the __fmul2_rn / __fadd2_rn intrinsics
// were contracted into FFMA2 by the compiler, which would change the reference's rounding).
__device__ __forceinline__ float2 mul2_rn(float2 a, float2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<const float2*>(&r);
}
__device__ __forceinline__ float2 add2_rn(float2 a, float2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<const float2*>(&r);
}

// Same arithmetic (per output: bias, then taps in (dt, df) order, then input channels, separately
// rounded products and sums, out-of-range taps skipped), PX horizontally adjacent output pixels per
// thread, so every weight read from shared memory feeds PX x 16 products instead of 16.
template <int PX>
__global__ void __launch_bounds__(128) conv_f32_px_kernel(const ConvF32 p) {
  extern __shared__ float sw[];  // [kh*kw][cin][kCot]
  const int co0 = blockIdx.y * kCot;
  const int ncot = min(kCot, p.cout - co0);
  const int taps = p.kh * p.kw;
  for (int i = threadIdx.x; i < taps * p.cin * kCot; i += blockDim.x) {
    const int co = i % kCot;
    const int tci = i / kCot;
    sw[i] = co < ncot ? p.w[static_cast<int64_t>(tci) * p.cout + co0 + co] : 0.f;
  }
  __syncthreads();
  const int64_t npix = static_cast<int64_t>(p.B) * p.T * p.F;
  const int64_t pix0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * PX;
  if (pix0 >= npix) return;
  int fk[PX], tk[PX];
  int64_t bk[PX];
  bool live[PX];
#pragma unroll
  for (int k = 0; k < PX; ++k) {
    const int64_t pix = pix0 + k;
    live[k] = pix < npix;
    fk[k] = static_cast<int>(pix % p.F);
    tk[k] = static_cast<int>((pix / p.F) % p.T);
    bk[k] = pix / (static_cast<int64_t>(p.F) * p.T);
  }
  float acc[PX][kCot];
#pragma unroll
  for (int k = 0; k < PX; ++k)
#pragma unroll
    for (int c = 0; c < kCot; ++c) acc[k][c] = (p.bias && c < ncot) ? p.bias[co0 + c] : 0.f;
  const int oh = p.kh / 2, ow = p.kw / 2;
  for (int dt = 0; dt < p.kh; ++dt) {
    for (int df = 0; df < p.kw; ++df) {
      const float* xr[PX];
      bool ok[PX];
      bool any = false;
#pragma unroll
      for (int k = 0; k < PX; ++k) {
        const int ti = tk[k] + dt - oh, fi = fk[k] + (df - ow) * p.dil_f;
        ok[k] = live[k] && ti >= 0 && ti < p.T && fi >= 0 && fi < p.F;
        xr[k] = p.x + ((bk[k] * p.T + (ok[k] ? ti : 0)) * p.F + (ok[k] ? fi : 0)) * p.cin;
        any |= ok[k];
      }
      if (!any) continue;
      const float* wt = sw + (dt * p.kw + df) * p.cin * kCot;
      int ci = 0;
      if ((p.cin & 3) == 0) {
        for (; ci < p.cin; ci += 4) {
          float4 xv[PX];
#pragma unroll
          for (int k = 0; k < PX; ++k) xv[k] = ok[k] ? *reinterpret_cast<const float4*>(xr[k] + ci) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4* w4 = reinterpret_cast<const float4*>(wt + (ci + u) * kCot);
            float4 wv[kCot / 4];
#pragma unroll
            for (int q = 0; q < kCot / 4; ++q) wv[q] = w4[q];
            // pixel pairs (k, k+1) with both taps in range: packed products (FMUL2), scalar sums
#pragma unroll
            for (int k = 0; k < PX; k += 2) {
              const float x0 = u == 0 ? xv[k].x : u == 1 ? xv[k].y : u == 2 ? xv[k].z : xv[k].w;
              const float x1 = u == 0 ? xv[k + 1].x : u == 1 ? xv[k + 1].y : u == 2 ? xv[k + 1].z : xv[k + 1].w;
              if (ok[k] && ok[k + 1]) {
                const float2 xs = make_float2(x0, x1);
#pragma unroll
                for (int q = 0; q < kCot / 4; ++q) {
                  const float wq[4] = {wv[q].x, wv[q].y, wv[q].z, wv[q].w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float2 m = mul2_rn(xs, make_float2(wq[e], wq[e]));
                    acc[k][4 * q + e] = __fadd_rn(acc[k][4 * q + e], m.x);
                    acc[k + 1][4 * q + e] = __fadd_rn(acc[k + 1][4 * q + e], m.y);
                  }
                }
              } else {
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                  if (!ok[k + kk]) continue;
                  const float xs = kk == 0 ? x0 : x1;
#pragma unroll
                  for (int q = 0; q < kCot / 4; ++q) {
                    acc[k + kk][4 * q + 0] = __fadd_rn(acc[k + kk][4 * q + 0], __fmul_rn(xs, wv[q].x));
                    acc[k + kk][4 * q + 1] = __fadd_rn(acc[k + kk][4 * q + 1], __fmul_rn(xs, wv[q].y));
                    acc[k + kk][4 * q + 2] = __fadd_rn(acc[k + kk][4 * q + 2], __fmul_rn(xs, wv[q].z));
                    acc[k + kk][4 * q + 3] = __fadd_rn(acc[k + kk][4 * q + 3], __fmul_rn(xs, wv[q].w));
                  }
                }
              }
            }
          }
        }
      }
      for (; ci < p.cin; ++ci) {
#pragma unroll
        for (int k = 0; k < PX; ++k) {
          if (!ok[k]) continue;
          const float xv = xr[k][ci];
#pragma unroll
          for (int c = 0; c < kCot; ++c) acc[k][c] = __fadd_rn(acc[k][c], __fmul_rn(xv, wt[ci * kCot + c]));
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < PX; ++k) {
    if (!live[k]) continue;
    const int64_t pix = pix0 + k;
    float* yr = p.y + pix * p.cout + co0;
    const float* orow = p.other ? p.other + pix * p.cout + co0 : nullptr;
#pragma unroll
    for (int c = 0; c < kCot; ++c) {
      if (c >= ncot) break;
      float v = acc[k][c];
      if (p.aff_s) v = __fadd_rn(__fmul_rn(v, p.aff_s[co0 + c]), p.aff_t[co0 + c]);
      if (p.relu) v = v > 0.f ? v : 0.f;
      if (p.other_op == 6) v = __fadd_rn(v, orow[c]);
      if (p.other_op == 7) v = __fmul_rn(v, orow[c]);
      yr[c] = v;
    }
  }
}

__global__ void dwconv_f32_kernel(const float* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                                  float* __restrict__ y, int B, int T, int F, int C, int kh, int kw) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n = static_cast<int64_t>(B) * T * F * C;
  if (i >= n) return;
  const int c = static_cast<int>(i % C);
  const int64_t pix = i / C;
  const int f = static_cast<int>(pix % F);
  const int t = static_cast<int>((pix / F) % T);
  const int64_t b = pix / (static_cast<int64_t>(F) * T);
  float acc = bias ? bias[c] : 0.f;
  for (int dt = 0; dt < kh; ++dt) {
    const int ti = t + dt - kh / 2;
    if (ti < 0 || ti >= T) continue;
    for (int df = 0; df < kw; ++df) {
      const int fi = f + df - kw / 2;
      if (fi < 0 || fi >= F) continue;
      acc = __fadd_rn(acc, __fmul_rn(x[((b * T + ti) * F + fi) * C + c], w[(dt * kw + df) * C + c]));
    }
  }
  y[i] = acc;
}

__global__ void affine_f32_kernel(const float* __restrict__ x, const float* __restrict__ s, const float* __restrict__ t,
                                  int relu, float* __restrict__ y, int64_t n, int C) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = static_cast<int>(i % C);
  float v = __fadd_rn(__fmul_rn(x[i], s[c]), t[c]);
  if (relu) v = v > 0.f ? v : 0.f;
  y[i] = v;
}

__global__ void relu_f32_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] > 0.f ? x[i] : 0.f;
}

__global__ void binary_f32_kernel(int op, const float* __restrict__ a, const float* __restrict__ b,
                                  float* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = op == 7 ? __fmul_rn(a[i], b[i]) : __fadd_rn(a[i], b[i]);
}

// layer_norm (norms.hpp:155-191): double statistics per position, like the reference.
__global__ void layernorm_f32_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                     const float* __restrict__ bb, float* __restrict__ y, int64_t rows, int C,
                                     double eps) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const float* xr = x + r * C;
  double sum = 0.0, sq = 0.0;
  for (int i = 0; i < C; ++i) {
    sum = __dadd_rn(sum, static_cast<double>(xr[i]));
    sq = __dadd_rn(sq, __dmul_rn(static_cast<double>(xr[i]), static_cast<double>(xr[i])));
  }
  const double m = __ddiv_rn(sum, static_cast<double>(C));
  double v = __dsub_rn(__ddiv_rn(sq, static_cast<double>(C)), __dmul_rn(m, m));
  if (v < 0) v = 0;
  const double istd = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(v, eps)));
  for (int i = 0; i < C; ++i) {
    const double z = __dmul_rn(__dmul_rn(__dsub_rn(static_cast<double>(xr[i]), m), istd), static_cast<double>(g[i]));
    y[r * C + i] = static_cast<float>(__dadd_rn(z, static_cast<double>(bb[i])));
  }
}

__global__ void concat_f32_kernel(const float* __restrict__ a, int ca, const float* __restrict__ b, int cb,
                                  float* __restrict__ y, int64_t rows) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int cc = ca + cb;
  if (i >= rows * cc) return;
  const int64_t r = i / cc;
  const int c = static_cast<int>(i % cc);
  y[i] = c < ca ? a[r * ca + c] : b[r * cb + (c - ca)];
}

inline unsigned nblk(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

const char* launch_conv_f32(const ConvF32& p, cudaStream_t s) {
  const int64_t npix = static_cast<int64_t>(p.B) * p.T * p.F;
  const size_t smem = sizeof(float) * p.kh * p.kw * p.cin * kCot;
  if (smem > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(conv_f32_kernel), static_cast<int>(smem));
  require(smem <= 227 * 1024, "fp32 conv weights tile exceeds shared memory");
  static const int px = std::getenv("CNRX_F32_PX") ? std::atoi(std::getenv("CNRX_F32_PX")) : 2;
  if (px == 4 && npix >= 4 * 148 * 128) {
    if (smem > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(conv_f32_px_kernel<4>), static_cast<int>(smem));
    dim3 grid4(nblk((npix + 3) / 4, 128), static_cast<unsigned>((p.cout + kCot - 1) / kCot));
    conv_f32_px_kernel<4><<<grid4, 128, smem, s>>>(p);
    CNRX_CUDA(cudaGetLastError());
    return "conv_f32_px_kernel<4>";
  }
  if (px >= 2 && npix >= 2 * 148 * 128) {
    if (smem > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(conv_f32_px_kernel<2>), static_cast<int>(smem));
    dim3 grid2(nblk((npix + 1) / 2, 128), static_cast<unsigned>((p.cout + kCot - 1) / kCot));
    conv_f32_px_kernel<2><<<grid2, 128, smem, s>>>(p);
    CNRX_CUDA(cudaGetLastError());
    return "conv_f32_px_kernel<2>";
  }
  dim3 grid(nblk(npix, 128), static_cast<unsigned>((p.cout + kCot - 1) / kCot));
  conv_f32_kernel<<<grid, 128, smem, s>>>(p);
  CNRX_CUDA(cudaGetLastError());
  return "conv_f32_kernel";
}

const char* launch_dwconv_f32(const float* x, const float* w, const float* bias, float* y, int B, int T, int F,
                              int C, int kh, int kw, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(B) * T * F * C;
  dwconv_f32_kernel<<<nblk(n, 256), 256, 0, s>>>(x, w, bias, y, B, T, F, C, kh, kw);
  CNRX_CUDA(cudaGetLastError());
  return "dwconv_f32_kernel";
}

const char* launch_affine_f32(const float* x, const float* s_, const float* t_, int relu, float* y, int64_t rows,
                              int C, cudaStream_t s) {
  affine_f32_kernel<<<nblk(rows * C, 256), 256, 0, s>>>(x, s_, t_, relu, y, rows * C, C);
  CNRX_CUDA(cudaGetLastError());
  return "affine_f32_kernel";
}

const char* launch_relu_f32(const float* x, float* y, int64_t n, cudaStream_t s) {
  relu_f32_kernel<<<nblk(n, 256), 256, 0, s>>>(x, y, n);
  CNRX_CUDA(cudaGetLastError());
  return "relu_f32_kernel";
}

const char* launch_binary_f32(int op, const float* a, const float* b, float* y, int64_t n, cudaStream_t s) {
  binary_f32_kernel<<<nblk(n, 256), 256, 0, s>>>(op, a, b, y, n);
  CNRX_CUDA(cudaGetLastError());
  return "binary_f32_kernel";
}

const char* launch_layernorm_f32(const float* x, const float* g, const float* b, float* y, int64_t rows, int C,
                                 double eps, cudaStream_t s) {
  layernorm_f32_kernel<<<nblk(rows, 128), 128, 0, s>>>(x, g, b, y, rows, C, eps);
  CNRX_CUDA(cudaGetLastError());
  return "layernorm_f32_kernel";
}

const char* launch_concat_f32(const float* a, int ca, const float* b, int cb, float* y, int64_t rows, cudaStream_t s) {
  concat_f32_kernel<<<nblk(rows * (ca + cb), 256), 256, 0, s>>>(a, ca, b, cb, y, rows);
  CNRX_CUDA(cudaGetLastError());
  return "concat_f32_kernel";
}

}  // namespace cnrx
