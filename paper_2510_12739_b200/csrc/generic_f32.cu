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

#include <algorithm>
#include <string>
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
// acc + m as fma.rn.f32x2(m, one, acc) with `one` a runtime 1.0 (a kernel argument): m * 1 is exact, so
// this is the separately rounded add; ptxas contracts a mul.rn.f32x2 feeding an add.rn.f32x2 into FFMA2
// (single rounding) even under -fmad=false, but cannot fold a product into an fma it cannot see through.
__device__ __forceinline__ float2 acc2_rn(float2 acc, float2 m, float2 one) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(*reinterpret_cast<const uint64_t*>(&m)), "l"(*reinterpret_cast<const uint64_t*>(&one)), "l"(*reinterpret_cast<const uint64_t*>(&acc)));
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

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}

// Row stride (words) of a staged input pixel: cin rounded up to 4 (16-byte reads of four channels), with
// an odd number of 16-byte units so the 8 lanes of each LDS.128 phase, walking f, hit distinct banks.
__host__ __device__ inline int f32_tile_row_stride(int cin) {
  const int u = (cin + 3) / 4;
  return 4 * (u | 1);
}

// Shared-memory tiled form of the same conv (same per-output operation order: bias, taps in (dt, df)
// order, input channels in order, separately rounded products and sums, out-of-range taps skipped).
// A block owns one slot's T x FT output window for NG x COT output channels: the T x (FT + 2*halo) x cin
// input window is staged in shared memory once (cp.async; row stride f32_tile_row_stride) and shared by NG groups of 128 threads, group g computing output channels
// [co0 + g*COT, +COT) from its own weight slab [tap][cin][COT].  A thread computes PX adjacent pixels
// of one row as COT/2 channel pairs: one packed multiply (mul.rn.f32x2) and one packed add per two MACs,
// each lane rounded on its own — the reference's scalar x*w then y+=, two at a time.  (Packing saves
// issue slots only: the FP32 pipe does 128 lane-ops/clk/SM either way, tools/probes/ffma2_probe.cu.)
template <int PX, int COT, int NG, bool WS>
__global__ void __launch_bounds__(128 * NG) conv_f32_tile_kernel(const ConvF32 p, int FT, int ntf, float one_) {
  const float2 one = make_float2(one_, one_);
  extern __shared__ __align__(16) float smem_f[];
  const int taps = p.kh * p.kw;
  const int oh = p.kh / 2, ow = p.kw / 2;
  const int hf = ow * p.dil_f;
  const int W = FT + 2 * hf;
  const int cs = f32_tile_row_stride(p.cin);
  const int wtap = p.cin * COT;                 // one group's weights of one tap: [cin][COT]
  const int wslab = (WS ? 1 : taps) * wtap;     // one group's share of a weight buffer
  float* sx = smem_f + (WS ? 2 : 1) * NG * wslab;  // [T][W][cs] after the weight buffer(s) [NG][taps|1][cin][COT]
  const int b = blockIdx.x / ntf;
  const int f0 = (blockIdx.x % ntf) * FT;
  const int cob = blockIdx.y * NG * COT;
  // staging by cp.async (4-byte copies, zero-filled when out of range): every load in flight at once
  auto stage_w = [&](int tap0, int ntap, float* dst) {
    for (int i = threadIdx.x; i < NG * ntap * wtap; i += blockDim.x) {
      const int gi = i / (ntap * wtap), r = i - gi * ntap * wtap;
      const int co = cob + gi * COT + r % COT;
      const int tci = tap0 * p.cin + r / COT;  // tap * cin + ci
      cp_async4(dst + i, p.w + static_cast<int64_t>(tci) * p.cout + (co < p.cout ? co : 0), co < p.cout);
    }
  };
  stage_w(0, WS ? 1 : taps, smem_f);
  {
    const float* xb = p.x + static_cast<int64_t>(b) * p.T * p.F * p.cin;
    // one warp per window pixel, lanes over its channels (coalesced: a pixel's cin floats are contiguous)
    const int lane = threadIdx.x & 31;
    for (int pc = threadIdx.x >> 5; pc < p.T * W; pc += blockDim.x >> 5) {
      const int t = pc / W, fc = pc - t * W;
      const int fi = f0 - hf + fc;
      const bool in = fi >= 0 && fi < p.F;
      const float* src = xb + (static_cast<int64_t>(t) * p.F + (in ? fi : 0)) * p.cin;
      for (int ci = lane; ci < p.cin; ci += 32) cp_async4(sx + pc * cs + ci, src + ci, in);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  const int g = threadIdx.x / 128;
  const int co0 = cob + g * COT;
  const int ncot = min(COT, p.cout - co0);
  const int tid = threadIdx.x % 128;
  const int tpr = FT / PX;
  const int t = tid / tpr;
  const int fl = (tid - t * tpr) * PX;  // first local column of this thread
  const bool active = ncot > 0 && t < p.T && f0 + fl < p.F;
  if (!WS && !active) return;  // (streamed weights: every thread stays for the per-tap barriers)
  bool live[PX];
#pragma unroll
  for (int k = 0; k < PX; ++k) live[k] = f0 + fl + k < p.F;
  float2 acc[PX][COT / 2];
#pragma unroll
  for (int k = 0; k < PX; ++k)
#pragma unroll
    for (int q = 0; q < COT / 2; ++q)
      acc[k][q] = make_float2((active && p.bias && 2 * q < ncot) ? p.bias[co0 + 2 * q] : 0.f,
                              (active && p.bias && 2 * q + 1 < ncot) ? p.bias[co0 + 2 * q + 1] : 0.f);
  for (int tap = 0; tap < taps; ++tap) {
    if (WS && tap + 1 < taps) stage_w(tap + 1, 1, smem_f + ((tap + 1) & 1) * NG * wslab);
    const int dt = tap / p.kw, df = tap - dt * p.kw;
    const int ti = t + dt - oh;
    bool ok[PX];
    bool all = true, any = false;
#pragma unroll
    for (int k = 0; k < PX; ++k) {
      const int fi = f0 + fl + k + (df - ow) * p.dil_f;
      ok[k] = active && live[k] && ti >= 0 && ti < p.T && fi >= 0 && fi < p.F;
      all &= ok[k];
      any |= ok[k];
    }
    if (any) {
      const float* xr = sx + (ti * W + fl + df * p.dil_f) * cs;  // pixel k at xr + k*cs
      const float* wt = WS ? smem_f + (tap & 1) * NG * wslab + g * wslab : smem_f + g * wslab + tap * wtap;
      if (all) {
        // four input channels per step: one 16-byte read of each pixel's x, 4 x COT/4 of weights
        const int cin4 = p.cin >> 2;
#pragma unroll 2
        for (int c4 = 0; c4 < cin4; ++c4) {
          float4 xq[PX];
#pragma unroll
          for (int k = 0; k < PX; ++k) xq[k] = *reinterpret_cast<const float4*>(xr + k * cs + 4 * c4);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4* w4 = reinterpret_cast<const float4*>(wt + (4 * c4 + u) * COT);
            float2 wp[COT / 2];
#pragma unroll
            for (int q = 0; q < COT / 4; ++q) {
              const float4 v = w4[q];
              wp[2 * q] = make_float2(v.x, v.y);
              wp[2 * q + 1] = make_float2(v.z, v.w);
            }
#pragma unroll
            for (int k = 0; k < PX; ++k) {
              const float xv = u == 0 ? xq[k].x : u == 1 ? xq[k].y : u == 2 ? xq[k].z : xq[k].w;
              const float2 xx = make_float2(xv, xv);
#pragma unroll
              for (int q = 0; q < COT / 2; ++q) acc[k][q] = acc2_rn(acc[k][q], mul2_rn(xx, wp[q]), one);
            }
          }
        }
        for (int ci = 4 * cin4; ci < p.cin; ++ci) {
          const float4* w4 = reinterpret_cast<const float4*>(wt + ci * COT);
          float2 wp[COT / 2];
#pragma unroll
          for (int q = 0; q < COT / 4; ++q) {
            const float4 v = w4[q];
            wp[2 * q] = make_float2(v.x, v.y);
            wp[2 * q + 1] = make_float2(v.z, v.w);
          }
#pragma unroll
          for (int k = 0; k < PX; ++k) {
            const float xv = xr[k * cs + ci];
            const float2 xx = make_float2(xv, xv);
#pragma unroll
            for (int q = 0; q < COT / 2; ++q) acc[k][q] = acc2_rn(acc[k][q], mul2_rn(xx, wp[q]), one);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < PX; ++k) {
          if (!ok[k]) continue;
          for (int ci = 0; ci < p.cin; ++ci) {
            const float4* w4 = reinterpret_cast<const float4*>(wt + ci * COT);
            const float xv = xr[k * cs + ci];
            const float2 xx = make_float2(xv, xv);
#pragma unroll
            for (int q = 0; q < COT / 4; ++q) {
              const float4 v = w4[q];
              acc[k][2 * q] = acc2_rn(acc[k][2 * q], mul2_rn(xx, make_float2(v.x, v.y)), one);
              acc[k][2 * q + 1] = acc2_rn(acc[k][2 * q + 1], mul2_rn(xx, make_float2(v.z, v.w)), one);
            }
          }
        }
      }
    }
    if (WS) {
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
  }
  if (!active) return;
  const int64_t pixrow = (static_cast<int64_t>(b) * p.T + t) * p.F + f0 + fl;
#pragma unroll
  for (int k = 0; k < PX; ++k) {
    if (!live[k]) continue;
    const int64_t pix = pixrow + k;
    float* yr = p.y + pix * p.cout + co0;
    const float* orow = p.other ? p.other + pix * p.cout + co0 : nullptr;
    float v[COT];
#pragma unroll
    for (int c = 0; c < COT; ++c) {
      v[c] = (c & 1) ? acc[k][c / 2].y : acc[k][c / 2].x;
      if (c >= ncot) continue;
      if (p.aff_s) v[c] = __fadd_rn(__fmul_rn(v[c], p.aff_s[co0 + c]), p.aff_t[co0 + c]);
      if (p.relu) v[c] = v[c] > 0.f ? v[c] : 0.f;
      if (p.other_op == 6) v[c] = __fadd_rn(v[c], orow[c]);
      if (p.other_op == 7) v[c] = __fmul_rn(v[c], orow[c]);
    }
    if (ncot == COT && (p.cout & 3) == 0) {
#pragma unroll
      for (int c = 0; c < COT; c += 4) *reinterpret_cast<float4*>(yr + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
    } else {
#pragma unroll
      for (int c = 0; c < COT; ++c)
        if (c < ncot) yr[c] = v[c];
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

// T rows x FT columns per block, PX pixels per thread; NG groups x COT output channels share the staged
// input window.  Returns null when the window does not fit (the caller falls back to conv_f32_px).
// T rows x FT columns per block, PX pixels per thread; NG groups x COT output channels share the staged
// input window.  Weights: all taps resident, or (WS) one tap at a time, double-buffered, when the
// resident form would leave fewer than two blocks per SM (force_ws: -1 choose, 0 resident only, 1 WS).
// Returns null when that does not fit (the caller falls back to conv_f32_px).
template <int PX, int COT, int NG>
const char* launch_conv_f32_tile(const ConvF32& p, cudaStream_t s, int force_ws = -1) {
  int FT = (128 / p.T) * PX;
  FT = std::min(FT, (p.F + PX - 1) / PX * PX);
  const int hf = (p.kw / 2) * p.dil_f;
  const size_t xwin = static_cast<size_t>(p.T) * (FT + 2 * hf) * f32_tile_row_stride(p.cin);
  const size_t wres = static_cast<size_t>(NG) * p.kh * p.kw * p.cin * COT;
  const size_t wstr = 2 * static_cast<size_t>(NG) * p.cin * COT;
  // resident weights while two blocks still fit on an SM (2 x (112 + 1 reserved) KB of 228)
  const bool fits2 = sizeof(float) * (wres + xwin) <= 112 * 1024;
  if (force_ws == 0 && !fits2) return nullptr;
  const bool ws = force_ws >= 0 ? force_ws == 1 : !fits2;
  const size_t tsmem = sizeof(float) * ((ws ? wstr : wres) + xwin);
  if (tsmem > 200 * 1024) return nullptr;
  const int ntf = (p.F + FT - 1) / FT;
  auto kern = ws ? conv_f32_tile_kernel<PX, COT, NG, true> : conv_f32_tile_kernel<PX, COT, NG, false>;
  if (tsmem > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(tsmem));
  dim3 grid(static_cast<unsigned>(p.B * ntf), static_cast<unsigned>((p.cout + NG * COT - 1) / (NG * COT)));
  kern<<<grid, 128 * NG, tsmem, s>>>(p, FT, ntf, 1.0f);
  CNRX_CUDA(cudaGetLastError());
  static const std::string name[2] = {
      "conv_f32_tile_kernel<" + std::to_string(PX) + "," + std::to_string(COT) + "," + std::to_string(NG) + ">",
      "conv_f32_tile_kernel<" + std::to_string(PX) + "," + std::to_string(COT) + "," + std::to_string(NG) + ",ws>"};
  return name[ws].c_str();
}

const char* launch_conv_f32(const ConvF32& p, cudaStream_t s) {
  const int64_t npix = static_cast<int64_t>(p.B) * p.T * p.F;
  const size_t smem = sizeof(float) * p.kh * p.kw * p.cin * kCot;
  require(smem <= 227 * 1024, "fp32 conv weights tile exceeds shared memory");
  if (smem > 48 * 1024) ensure_smem_attr(reinterpret_cast<const void*>(conv_f32_kernel), static_cast<int>(smem));
  static const int px = std::getenv("CNRX_F32_PX") ? std::atoi(std::getenv("CNRX_F32_PX")) : 2;
  static const int tile = std::getenv("CNRX_F32_TILE") ? std::atoi(std::getenv("CNRX_F32_TILE")) : 1;
  if (tile && p.T <= 64) {
    switch (tile) {  // 1: measured choice (tools/f32_ab.py, profiles/r02_f32_tile_ab.log); 2..8 A/B variants
      case 2: if (const char* n = launch_conv_f32_tile<1, 8, 2>(p, s)) return n; break;
      case 3: if (const char* n = launch_conv_f32_tile<2, 8, 4>(p, s)) return n; break;
      case 4: if (const char* n = launch_conv_f32_tile<2, 8, 2>(p, s, 1)) return n; break;
      case 5: if (const char* n = launch_conv_f32_tile<1, 8, 4>(p, s)) return n; break;
      case 6: if (const char* n = launch_conv_f32_tile<1, 16, 2>(p, s)) return n; break;
      case 7: if (const char* n = launch_conv_f32_tile<1, 8, 2>(p, s, 1)) return n; break;
      case 8: if (const char* n = launch_conv_f32_tile<2, 8, 4>(p, s, 1)) return n; break;
      default:
        // narrow inputs (cfg1's 32 channels): one pixel per thread, twice the warps; wide inputs: two
        // pixels per thread (half the weight reads) while the weights stay resident, else one pixel per
        // thread with per-tap weights (96 channels: 13.1 -> 9.6 ms for cfg4 B = 8)
        if (p.cin > 32)
          if (const char* n = launch_conv_f32_tile<2, 8, 2>(p, s, 0)) return n;
        if (const char* n = launch_conv_f32_tile<1, 8, 2>(p, s)) return n;
        break;
    }
  }
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
