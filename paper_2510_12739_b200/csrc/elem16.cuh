// elem16.cuh — the two 16-bit activation/weight formats of the tensor-core plans.
//
// CNRX_BF16 plans store every activation plane and every conv weight as bf16 (8-bit mantissa);
// CNRX_FP16 plans store them as IEEE fp16 (11-bit mantissa, |x| <= 65504).  Both feed the same
// tcgen05 kind::f16 UMMAs with fp32 accumulation at the same rate and move the same bytes; only the
// instruction descriptor's operand-format fields and the pack/unpack instructions differ, so every
// tensor-core kernel is written once over `bool H` (H = fp16).  fp16 packs saturate to the largest
// finite value (cvt.rn.satfinite) instead of overflowing to inf.
//
// Why fp16 exists: on the trained cfg2 checkpoint no placement of bf16 roundings
// reaches the north star's 99.99 % hard-decision agreement with the fp32 reference — even bf16 conv
// operands alone (everything else fp32) leave 99.987 % (tools/ablate_bf16.py, profiles/r02_ablate_bf16.jsonl);
// the same plan in fp16 reaches 99.993 %.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <cstring>

namespace cnrx {

// tcgen05 instruction-descriptor operand format (kind::f16): 0 = f16, 1 = bf16
template <bool H>
__host__ __device__ constexpr uint32_t e16_fmt() {
  return H ? 0u : 1u;
}
// D = f32, A/B = the plan's 16-bit format, both K-major, M x N
template <bool H>
__host__ __device__ constexpr uint32_t idesc_e16_f32(uint32_t M, uint32_t N) {
  return (1u << 4) | (e16_fmt<H>() << 7) | (e16_fmt<H>() << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

#ifdef __CUDACC__
// (lo, hi) -> packed pair, lo in the low half (the element at the lower address)
template <bool H>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  uint32_t r;
  if constexpr (H)
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  else
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
template <bool H>
__device__ __forceinline__ float2 unpack2(uint32_t u) {
  if constexpr (H) {
    __half2 h;
    std::memcpy(&h, &u, 4);
    return __half22float2(h);
  } else {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
  }
}
// max(x, 0) on both halves
template <bool H>
__device__ __forceinline__ uint32_t relu2(uint32_t u) {
  uint32_t r;
  if constexpr (H)
    asm("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(u), "r"(0u));
  else
    asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(u), "r"(0u));
  return r;
}
// runtime-format forms for the HBM-bound kernels (featurize, pointwise programs, head): one uniform
// branch per pair
__device__ __forceinline__ uint32_t pack2r(bool h, float lo, float hi) { return h ? pack2<true>(lo, hi) : pack2<false>(lo, hi); }
__device__ __forceinline__ float2 unpack2r(bool h, uint32_t u) { return h ? unpack2<true>(u) : unpack2<false>(u); }
__device__ __forceinline__ uint32_t relu2r(bool h, uint32_t u) { return h ? relu2<true>(u) : relu2<false>(u); }
#endif

// host: fp32 -> 16-bit bits (weights at plan creation), round to nearest even; fp16 saturates
inline uint16_t e16_from_float_host(float v, bool h) {
  uint16_t bits;
  if (h) {
    const float lim = 65504.f;
    const __half x = __float2half_rn(v > lim ? lim : (v < -lim ? -lim : v));
    std::memcpy(&bits, &x, 2);
  } else {
    const __nv_bfloat16 x = __float2bfloat16(v);
    std::memcpy(&bits, &x, 2);
  }
  return bits;
}
inline float e16_to_float_host(uint16_t bits, bool h) {
  if (h) {
    __half x;
    std::memcpy(&x, &bits, 2);
    return __half2float(x);
  }
  const uint32_t u = static_cast<uint32_t>(bits) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

}  // namespace cnrx
