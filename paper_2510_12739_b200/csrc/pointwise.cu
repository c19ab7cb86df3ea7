// pointwise.cu — linear pointwise programs over bf16 planes: the CoNet interaction + post-fusion BN
// chain and the 1x1 LLR head (network.hpp:534-559: mul -> norm -> ... -> main.out conv), or any
// non-conv pointwise node the plan compiler has to materialise as a plane.
//
// One thread per plane row; the row's C channels are processed in 8-channel slices (one 16-byte load
// per operand plane per slice).  The head GEMV (C -> bits, fp32) runs on CUDA cores from a shared-memory
// copy of the head weights; LLRs are written in the reference layout [B,T,F,bits] (fp32), so padding
// rows produce no output.  HBM-bound: it reads C*2 bytes per operand plane and writes 4*bits bytes.
#include <cuda_runtime.h>

#include "kernels.h"

namespace cnrx {

namespace {

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

template <int HEAD>
__global__ void __launch_bounds__(256) pw_program_kernel(const __grid_constant__ PwProgram prog, PlaneGeom geo) {
  extern __shared__ float s_head[];  // [C][bits] + [bits]
  const int C = prog.C, NB = prog.head_bits;
  if (HEAD) {
    for (int i = threadIdx.x; i < C * NB; i += blockDim.x) s_head[i] = prog.head_w[i];
    for (int i = threadIdx.x; i < NB; i += blockDim.x) s_head[C * NB + i] = prog.head_b[i];
    __syncthreads();
  }
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= geo.Nalloc) return;
  const bool valid = geo.valid(row);
  if (HEAD && !valid) return;
  float out[kPwMaxBits];
  if (HEAD) {
#pragma unroll
    for (int j = 0; j < kPwMaxBits; ++j) out[j] = 0.f;
  }
  for (int c0 = 0; c0 < C; c0 += 8) {
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    if (valid) {
      for (int n = 0; n < prog.n_ins; ++n) {
        const PwIns ins = prog.ins[n];
        if (ins.op == PW_LOAD || ins.op == PW_MUL || ins.op == PW_ADD) {
          float v[8];
          load8(prog.planes[ins.k] + row * C + c0, v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            acc[i] = ins.op == PW_LOAD ? v[i] : ins.op == PW_MUL ? acc[i] * v[i] : acc[i] + v[i];
        } else if (ins.op == PW_AFF) {
          const float* s = prog.aff_s[ins.k];
          const float* t = prog.aff_t[ins.k];
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = acc[i] * __ldg(&s[c0 + i]) + __ldg(&t[c0 + i]);
        } else {  // PW_RELU
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fmaxf(acc[i], 0.f);
        }
      }
    }
    if (HEAD) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float* wr = s_head + (c0 + i) * NB;
#pragma unroll
        for (int j = 0; j < kPwMaxBits; ++j)
          if (j < NB) out[j] += acc[i] * wr[j];
      }
    } else {
      uint4 o;
      __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) op[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      *reinterpret_cast<uint4*>(prog.out_plane + row * C + c0) = o;
    }
  }
  if (HEAD) {
    int b, t, f;
    geo.coords(row, b, t, f);
    float* dst = prog.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * NB;
#pragma unroll
    for (int j = 0; j < kPwMaxBits; ++j)
      if (j < NB) dst[j] = out[j] + s_head[C * NB + j];
  }
}

}  // namespace

const char* launch_pw_program(const PwProgram& prog, const PlaneGeom& geo, cudaStream_t s) {
  const int threads = 256;
  const unsigned blocks = static_cast<unsigned>((geo.Nalloc + threads - 1) / threads);
  if (prog.head_bits > 0) {
    require(prog.head_bits <= kPwMaxBits, "head with more than 16 outputs");
    const size_t smem = sizeof(float) * (static_cast<size_t>(prog.C) * prog.head_bits + prog.head_bits);
    pw_program_kernel<1><<<blocks, threads, smem, s>>>(prog, geo);
    CNRX_CUDA(cudaGetLastError());
    return "pw_program_kernel<head>";
  }
  pw_program_kernel<0><<<blocks, threads, 0, s>>>(prog, geo);
  CNRX_CUDA(cudaGetLastError());
  return "pw_program_kernel<plane>";
}

}  // namespace cnrx
