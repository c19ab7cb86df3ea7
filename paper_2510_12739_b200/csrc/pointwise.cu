// pointwise.cu — linear pointwise programs over 16-bit (bf16 / fp16) planes: the CoNet interaction + post-fusion BN
// chain and the 1x1 LLR head (network.hpp:534-559: mul -> norm -> ... -> main.out conv), or any
// non-conv pointwise node the plan compiler has to materialise as a plane.
//
// One thread per plane row; the row's C channels are processed in 8-channel slices (one 16-byte load
// per operand plane per slice).  The head GEMV (C -> bits, fp32) runs on CUDA cores from a shared-memory
// copy of the head weights; LLRs are written in the reference layout [B,T,F,bits] (fp32), so padding
// rows produce no output.  HBM-bound: it reads C*2 bytes per operand plane and writes 4*bits bytes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "head.h"
#include "kernels.h"
#include "elem16.cuh"

namespace cnrx {

namespace {

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&v)[8], bool h16) {
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  const uint32_t* h = reinterpret_cast<const uint32_t*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = unpack2r(h16, h[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

// 8 values -> (hi, lo) 16-bit halves of a split-plane row (hi at p, lo at p + C)
__device__ __forceinline__ void store8_split(__nv_bfloat16* p, int C, const float (&v)[8], bool h16) {
  uint4 oh, ol;
  uint32_t* ph = reinterpret_cast<uint32_t*>(&oh);
  uint32_t* pl = reinterpret_cast<uint32_t*>(&ol);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ph[i] = pack2r(h16, v[2 * i], v[2 * i + 1]);
    const float2 f = unpack2r(h16, ph[i]);
    pl[i] = pack2r(h16, v[2 * i] - f.x, v[2 * i + 1] - f.y);
  }
  *reinterpret_cast<uint4*>(p) = oh;
  *reinterpret_cast<uint4*>(p + C) = ol;
}

// Layer-norm programs (prog.ln = k + 1, plane output): the chain for all C channels of the row into local
// memory, then norms.hpp:171-184's statistics in double (sum and sum of squares, v = sq / c - m^2 clamped at
// 0, istd = 1 / sqrt(v + eps)) over the real channels, y = (x - m) * istd * g + b in double, then the
// 16-bit (or split) store; padding channels and invalid rows stay 0.
constexpr int kLnMaxC = 128;
constexpr double kPwLnEps = 1e-5;  // network.hpp:431
__global__ void __launch_bounds__(128) pw_ln_kernel(const __grid_constant__ PwProgram prog, PlaneGeom geo) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= geo.Nalloc) return;
  const int C = prog.C;
  const bool split = prog.split != 0, h16 = prog.fp16 != 0;
  const int64_t rs = split ? 2 * C : C;
  float acc[kLnMaxC];
  const bool valid = geo.valid(row);
  for (int c0 = 0; c0 < C; c0 += 8) {
    float a8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a8[i] = 0.f;
    if (valid) {
      for (int n = 0; n < prog.n_ins; ++n) {
        const PwIns ins = prog.ins[n];
        if (ins.op == PW_LOAD || ins.op == PW_MUL || ins.op == PW_ADD) {
          float v[8];
          load8(prog.planes[ins.k] + row * rs + c0, v, h16);
          if (split) {
            float l[8];
            load8(prog.planes[ins.k] + row * rs + C + c0, l, h16);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += l[i];
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
            a8[i] = ins.op == PW_LOAD ? v[i] : ins.op == PW_MUL ? a8[i] * v[i] : a8[i] + v[i];
        } else if (ins.op == PW_AFF) {
#pragma unroll
          for (int i = 0; i < 8; ++i) a8[i] = a8[i] * __ldg(&prog.aff_s[ins.k][c0 + i]) + __ldg(&prog.aff_t[ins.k][c0 + i]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) a8[i] = fmaxf(a8[i], 0.f);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[c0 + i] = a8[i];
  }
  const int k = prog.ln - 1, n = prog.ln_c;
  double sum = 0.0, sq = 0.0;
  for (int i = 0; i < n; ++i) {
    sum += acc[i];
    sq += static_cast<double>(acc[i]) * acc[i];
  }
  const double m = sum / n;
  double var = sq / n - m * m;
  if (var < 0) var = 0;
  const double istd = 1.0 / sqrt(var + kPwLnEps);
  for (int c0 = 0; c0 < C; c0 += 8) {
    float y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + i;
      y[i] = valid && c < n ? static_cast<float>((static_cast<double>(acc[c]) - m) * istd * prog.aff_s[k][c] + prog.aff_t[k][c])
                            : 0.f;
    }
    if (split) {
      store8_split(prog.out_plane + row * rs + c0, C, y, h16);
    } else {
      uint4 o;
      uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) op[i] = pack2r(h16, y[2 * i], y[2 * i + 1]);
      *reinterpret_cast<uint4*>(prog.out_plane + row * C + c0) = o;
    }
  }
}

template <int HEAD>
__global__ void __launch_bounds__(256) pw_program_kernel(const __grid_constant__ PwProgram prog, PlaneGeom geo) {
  extern __shared__ float s_head[];  // [C][bits] + [bits]
  const int C = prog.C, NB = prog.head_bits;
  const bool split = prog.split != 0;
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
          if (split) {
            float l[8];
            load8(prog.planes[ins.k] + row * 2 * C + c0, v, prog.fp16 != 0);
            load8(prog.planes[ins.k] + row * 2 * C + C + c0, l, prog.fp16 != 0);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += l[i];  // hi + lo: exact in fp32
          } else {
            load8(prog.planes[ins.k] + row * C + c0, v, prog.fp16 != 0);
          }
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
    } else if (split) {
      store8_split(prog.out_plane + row * 2 * C + c0, C, acc, prog.fp16 != 0);
      if (prog.out2_plane) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaxf(acc[i], 0.f);
        store8_split(prog.out2_plane + row * 2 * C + c0, C, acc, prog.fp16 != 0);
      }
    } else {
      uint4 o;
      uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) op[i] = pack2r(prog.fp16 != 0, acc[2 * i], acc[2 * i + 1]);
      *reinterpret_cast<uint4*>(prog.out_plane + row * C + c0) = o;
      if (prog.out2_plane) {
#pragma unroll
        for (int i = 0; i < 4; ++i) op[i] = relu2r(prog.fp16 != 0, op[i]);  // relu commutes with the rounding
        *reinterpret_cast<uint4*>(prog.out2_plane + row * C + c0) = o;
      }
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

// Coalesced variant for C in {16, 32, 64, 128}: LPR = C/8 lanes share a row (each lane owns one
// 16-byte, 8-channel slice), so a warp instruction reads 32 consecutive 16-byte slices of 32/LPR rows.
// The head GEMV partial sums are reduced across the row's lanes with shuffles.
// SPLIT (CNRX_*X3 plans): rows are [hi C | lo C]; a lane loads its 8-channel slice of both halves (each
// warp instruction still covers whole 128-byte lines) and stores the result split the same way.
template <int HEAD, int LPR, bool SPLIT = false, int NPMAX = kPwMaxPlanes>
__global__ void __launch_bounds__(256) pw_rows_kernel(const __grid_constant__ PwProgram prog, PlaneGeom geo) {
  extern __shared__ float smem_f[];
  const int C = prog.C, NB = prog.head_bits;
  float* s_w = smem_f;                               // [C][NB]
  float* s_b = s_w + (HEAD ? C * NB : 0);            // [NB]
  float* s_aff = s_b + (HEAD ? ((NB + 3) & ~3) : 0); // [n_aff][2][C]
  int n_aff = 0;
  for (int n = 0; n < prog.n_ins; ++n)
    if (prog.ins[n].op == PW_AFF) n_aff = max(n_aff, prog.ins[n].k + 1);
  // Tables are stored with the lane's channel group (cg = c / 8) innermost so the LPR lanes of a row,
  // which read the same (i, j) for different cg, hit distinct banks:
  //   s_w[(i * NB + j) * LPR + cg] = W[8 cg + i][j],  s_aff[((2k + st) * 8 + i) * LPR + cg]
  if (HEAD) {
    for (int e = threadIdx.x; e < C * NB; e += blockDim.x) {
      const int c = e / NB, jj = e % NB;
      s_w[((c % 8) * NB + jj) * LPR + c / 8] = prog.head_w[e];
    }
    for (int e = threadIdx.x; e < NB; e += blockDim.x) s_b[e] = prog.head_b[e];
  }
  for (int e = threadIdx.x; e < n_aff * C; e += blockDim.x) {
    const int k = e / C, c = e % C;
    s_aff[((2 * k) * 8 + c % 8) * LPR + c / 8] = prog.aff_s[k][c];
    s_aff[((2 * k + 1) * 8 + c % 8) * LPR + c / 8] = prog.aff_t[k][c];
  }
  __syncthreads();
  constexpr int RPW = 32 / LPR;  // rows per warp pass
  constexpr int U = 2;  // row groups per iteration (loads of both issued before compute)
  const int64_t RS = SPLIT ? 2 * C : C;  // row stride (16-bit values)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane % LPR;
  const int c0 = cg * 8;
  const int np = prog.n_planes_used;
  const int64_t groups = (geo.Nalloc + RPW - 1) / RPW;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * 8;
  for (int64_t grp0 = (static_cast<int64_t>(blockIdx.x) * 8 + warp) * U; grp0 < groups; grp0 += wstride * U) {
    int64_t row[U];
    bool in_range[U], valid[U];
    uint4 raw[U][NPMAX];
    uint4 rawl[U][SPLIT ? NPMAX : 1];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      row[u] = (grp0 + u) * RPW + lane / LPR;
      in_range[u] = row[u] < geo.Nalloc;
      valid[u] = in_range[u] && geo.valid(row[u]);
#pragma unroll
      for (int k = 0; k < NPMAX; ++k)
        if (k < np) {
          raw[u][k] = valid[u] ? *reinterpret_cast<const uint4*>(prog.planes[k] + row[u] * RS + c0)
                               : make_uint4(0, 0, 0, 0);
          if constexpr (SPLIT)
            rawl[u][k] = valid[u] ? *reinterpret_cast<const uint4*>(prog.planes[k] + row[u] * RS + C + c0)
                                  : make_uint4(0, 0, 0, 0);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float acc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.f;
      for (int n = 0; n < prog.n_ins; ++n) {
        const PwIns ins = prog.ins[n];
        if (ins.op == PW_LOAD || ins.op == PW_MUL || ins.op == PW_ADD) {
          uint4 r4 = raw[u][0];
#pragma unroll
          for (int k = 1; k < NPMAX; ++k)
            if (k == ins.k) r4 = raw[u][k];
          const uint32_t* h = reinterpret_cast<const uint32_t*>(&r4);
          float v[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = unpack2r(prog.fp16 != 0, h[i]);
            v[2 * i] = f.x;
            v[2 * i + 1] = f.y;
          }
          if constexpr (SPLIT) {
            uint4 l4 = rawl[u][0];
#pragma unroll
            for (int k = 1; k < NPMAX; ++k)
              if (k == ins.k) l4 = rawl[u][k];
            const uint32_t* hl = reinterpret_cast<const uint32_t*>(&l4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = unpack2r(prog.fp16 != 0, hl[i]);
              v[2 * i] += f.x;  // hi + lo: exact in fp32
              v[2 * i + 1] += f.y;
            }
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
            acc[i] = ins.op == PW_LOAD ? v[i] : ins.op == PW_MUL ? acc[i] * v[i] : acc[i] + v[i];
        } else if (ins.op == PW_AFF) {
          const float* sa = s_aff + (2 * ins.k) * 8 * LPR + cg;
          const float* ta = s_aff + (2 * ins.k + 1) * 8 * LPR + cg;
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = acc[i] * sa[i * LPR] + ta[i * LPR];
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fmaxf(acc[i], 0.f);
        }
      }
      if (!valid[u]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.f;
      }
      if (HEAD) {
        float part[kPwMaxBits];
#pragma unroll
        for (int j = 0; j < kPwMaxBits; ++j) part[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float* wr = s_w + (i * NB) * LPR + cg;
#pragma unroll
          for (int j = 0; j < kPwMaxBits; ++j)
            if (j < NB) part[j] += acc[i] * wr[j * LPR];
        }
#pragma unroll
        for (int off = LPR / 2; off >= 1; off >>= 1)
#pragma unroll
          for (int j = 0; j < kPwMaxBits; ++j)
            if (j < NB) part[j] += __shfl_xor_sync(0xffffffffu, part[j], off);
        if (valid[u] && cg == 0) {
          int b, t, f;
          geo.coords(row[u], b, t, f);
          float* dst = prog.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * NB;
          if (NB == 4) {
            *reinterpret_cast<float4*>(dst) = make_float4(part[0] + s_b[0], part[1] + s_b[1], part[2] + s_b[2],
                                                          part[3] + s_b[3]);
          } else {
#pragma unroll
            for (int j = 0; j < kPwMaxBits; ++j)
              if (j < NB) dst[j] = part[j] + s_b[j];
          }
        }
      } else if (in_range[u]) {
        if constexpr (SPLIT) {
          store8_split(prog.out_plane + row[u] * RS + c0, C, acc, prog.fp16 != 0);
        } else {
          uint4 o;
          uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
          for (int i = 0; i < 4; ++i) op[i] = pack2r(prog.fp16 != 0, acc[2 * i], acc[2 * i + 1]);
          *reinterpret_cast<uint4*>(prog.out_plane + row[u] * C + c0) = o;
        }
      }
    }
  }
}


// Fold kernel: LPR = C/8 lanes per row (lane cg owns channels [8cg, 8cg+8)); all NS operand loads of
// the row are issued before any arithmetic; BN tables and head weights are read from shared memory
// laid out [.][cg][8] so the lanes of a row read distinct banks and rows of a warp broadcast.
struct FoldSteps {
  int32_t op[kPwMaxPlanes];    // PW_MUL / PW_ADD for steps >= 1
  int32_t aff[kPwMaxPlanes];   // affine table index or -1
  int32_t relu[kPwMaxPlanes];
};

template <int HEAD, int LPR, int NS>
__global__ void __launch_bounds__(256) pw_fold_kernel(const __grid_constant__ PwProgram prog, const FoldSteps fs,
                                                      PlaneGeom geo) {
  extern __shared__ float smem_f[];
  constexpr int C = LPR * 8;
  constexpr int NB = HEAD;  // LLR outputs per RE (0: the program stores a plane)
  float* s_aff = smem_f;                              // [NS][2][LPR][8]
  float* s_w = s_aff + NS * 2 * C;                    // [8][NB][LPR]
  float* s_b = s_w + C * NB;                          // [NB]
  for (int e = threadIdx.x; e < NS * C; e += blockDim.x) {
    const int i = e / C, c = e % C;
    const int a = fs.aff[i];
    s_aff[(i * 2) * C + c] = a >= 0 ? prog.aff_s[a][c] : 1.f;
    s_aff[(i * 2 + 1) * C + c] = a >= 0 ? prog.aff_t[a][c] : 0.f;
  }
  if (NB > 0) {
    for (int e = threadIdx.x; e < C * NB; e += blockDim.x) {  // [e][j][cg]: lanes of a row hit distinct banks
      const int c = e / NB, j = e % NB;
      s_w[((c % 8) * NB + j) * LPR + c / 8] = prog.head_w[e];
    }
    for (int e = threadIdx.x; e < NB; e += blockDim.x) s_b[e] = prog.head_b[e];
  }
  __syncthreads();
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cg = lane % LPR;
  const int c0 = cg * 8;
  const int64_t groups = (geo.Nalloc + RPW - 1) / RPW;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * 8;
  constexpr int U = 4;  // row groups per warp iteration: U * NS 16-byte loads in flight per lane
  for (int64_t grp0 = (static_cast<int64_t>(blockIdx.x) * 8 + warp) * U; grp0 < groups; grp0 += wstride * U) {
    int64_t row[U];
    bool in_range[U], valid[U];
    uint4 raw[U][NS];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      row[u] = (grp0 + u) * RPW + lane / LPR;
      in_range[u] = row[u] < geo.Nalloc;
      valid[u] = in_range[u] && geo.valid(row[u]);
#pragma unroll
      for (int i = 0; i < NS; ++i)
        raw[u][i] = valid[u] ? __ldg(reinterpret_cast<const uint4*>(prog.planes[i] + row[u] * C + c0))
                             : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float acc[8];
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const uint32_t* h = reinterpret_cast<const uint32_t*>(&raw[u][i]);
        float v[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = unpack2r(prog.fp16 != 0, h[e]);
          v[2 * e] = f.x;
          v[2 * e + 1] = f.y;
        }
        if (i == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = v[e];
        } else if (fs.op[i] == PW_MUL) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] *= v[e];
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] += v[e];
        }
        if (fs.aff[i] >= 0) {
          const float4 s0 = *reinterpret_cast<const float4*>(s_aff + (i * 2) * C + c0);
          const float4 s1 = *reinterpret_cast<const float4*>(s_aff + (i * 2) * C + c0 + 4);
          const float4 t0 = *reinterpret_cast<const float4*>(s_aff + (i * 2 + 1) * C + c0);
          const float4 t1 = *reinterpret_cast<const float4*>(s_aff + (i * 2 + 1) * C + c0 + 4);
          acc[0] = acc[0] * s0.x + t0.x;
          acc[1] = acc[1] * s0.y + t0.y;
          acc[2] = acc[2] * s0.z + t0.z;
          acc[3] = acc[3] * s0.w + t0.w;
          acc[4] = acc[4] * s1.x + t1.x;
          acc[5] = acc[5] * s1.y + t1.y;
          acc[6] = acc[6] * s1.z + t1.z;
          acc[7] = acc[7] * s1.w + t1.w;
        }
        if (fs.relu[i]) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaxf(acc[e], 0.f);
        }
      }
      if constexpr (NB > 0) {
        float part[NB > 0 ? NB : 1];
#pragma unroll
        for (int j = 0; j < NB; ++j) part[j] = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float* wr = s_w + (e * NB) * LPR + cg;
#pragma unroll
          for (int j = 0; j < NB; ++j) part[j] = fmaf(acc[e], wr[j * LPR], part[j]);
        }
#pragma unroll
        for (int off = LPR / 2; off >= 1; off >>= 1)
#pragma unroll
          for (int j = 0; j < NB; ++j) part[j] += __shfl_xor_sync(0xffffffffu, part[j], off);
        if (valid[u] && cg == 0) {
          int b, t, f;
          geo.coords(row[u], b, t, f);
          float* dst = prog.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * NB;
          if constexpr (NB == 4) {
            *reinterpret_cast<float4*>(dst) =
                make_float4(part[0] + s_b[0], part[1] + s_b[1], part[2] + s_b[2], part[3] + s_b[3]);
          } else if constexpr (NB == 2) {
            *reinterpret_cast<float2*>(dst) = make_float2(part[0] + s_b[0], part[1] + s_b[1]);
          } else {
#pragma unroll
            for (int j = 0; j < NB; ++j) dst[j] = part[j] + s_b[j];
          }
        }
      } else if (in_range[u]) {
        if (!valid[u]) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        }
        uint4 o;
        uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) op[e] = pack2r(prog.fp16 != 0, acc[2 * e], acc[2 * e + 1]);
        *reinterpret_cast<uint4*>(prog.out_plane + row[u] * C + c0) = o;
      }
    }
  }
}

template <int HEAD, int LPR, int NS>
void launch_fold_t(const PwProgram& prog, const FoldSteps& fs, const PlaneGeom& geo, cudaStream_t s) {
  constexpr int C = LPR * 8;
  const size_t smem = sizeof(float) * (NS * 2 * C + (HEAD ? C * HEAD + HEAD : 0));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (geo.Nalloc + (32 / LPR) - 1) / (32 / LPR);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((groups + 31) / 32, static_cast<int64_t>(sms) * 8));
  pw_fold_kernel<HEAD, LPR, NS><<<blocks, 256, smem, s>>>(prog, fs, geo);
  CNRX_CUDA(cudaGetLastError());
}

template <int HEAD, int LPR>
bool launch_fold_ns(const PwProgram& prog, const FoldSteps& fs, int ns, const PlaneGeom& geo, cudaStream_t s) {
  switch (ns) {
    case 1: launch_fold_t<HEAD, LPR, 1>(prog, fs, geo, s); return true;
    case 2: launch_fold_t<HEAD, LPR, 2>(prog, fs, geo, s); return true;
    case 3: launch_fold_t<HEAD, LPR, 3>(prog, fs, geo, s); return true;
    case 4: launch_fold_t<HEAD, LPR, 4>(prog, fs, geo, s); return true;
    default: return false;
  }
}

template <int HEAD>
bool launch_fold_c(const PwProgram& prog, const FoldSteps& fs, int ns, const PlaneGeom& geo, cudaStream_t s) {
  switch (prog.C) {
    case 16: return launch_fold_ns<HEAD, 2>(prog, fs, ns, geo, s);
    case 32: return launch_fold_ns<HEAD, 4>(prog, fs, ns, geo, s);
    case 64: return launch_fold_ns<HEAD, 8>(prog, fs, ns, geo, s);
    case 128: return launch_fold_ns<HEAD, 16>(prog, fs, ns, geo, s);
    default: return false;
  }
}

// HEAD = LLR outputs per RE (compile-time: the GEMV and its shuffle reduction are fully unrolled)
bool launch_fold_any(const PwProgram& prog, const FoldSteps& fs, int ns, const PlaneGeom& geo, cudaStream_t s) {
  switch (prog.head_bits) {
    case 0: return launch_fold_c<0>(prog, fs, ns, geo, s);
    case 1: return launch_fold_c<1>(prog, fs, ns, geo, s);
    case 2: return launch_fold_c<2>(prog, fs, ns, geo, s);
    case 4: return launch_fold_c<4>(prog, fs, ns, geo, s);
    case 6: return launch_fold_c<6>(prog, fs, ns, geo, s);
    case 8: return launch_fold_c<8>(prog, fs, ns, geo, s);
    default: return false;
  }
}

// Fold program storing a plane (any C, multiple of 8): one thread per (row, 8-channel chunk), so
// consecutive threads touch consecutive 16-byte chunks (fully coalesced) and small batches still fill
// the GPU; optionally also writes relu(result) as a second plane (the next block's pre-activation).
template <int NS>
__global__ void __launch_bounds__(256) pw_fold_plane_kernel(const __grid_constant__ PwProgram prog,
                                                            const FoldSteps fs, PlaneGeom geo) {
  const int CC = prog.C / 8;  // chunks per row
  const int64_t total = geo.Nalloc * CC;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / CC;
    const int c0 = static_cast<int>(i - row * CC) * 8;
    const bool valid = geo.valid(row);
    uint4 raw[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k)
      raw[k] = valid ? __ldg(reinterpret_cast<const uint4*>(prog.planes[k] + row * prog.C + c0)) : make_uint4(0, 0, 0, 0);
    float acc[8];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const uint32_t* h = reinterpret_cast<const uint32_t*>(&raw[k]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = unpack2r(prog.fp16 != 0, h[e]);
        if (k == 0) {
          acc[2 * e] = f.x;
          acc[2 * e + 1] = f.y;
        } else if (fs.op[k] == PW_MUL) {
          acc[2 * e] *= f.x;
          acc[2 * e + 1] *= f.y;
        } else {
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
      if (fs.aff[k] >= 0) {
        const float* sv = prog.aff_s[fs.aff[k]] + c0;
        const float* tv = prog.aff_t[fs.aff[k]] + c0;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = acc[e] * __ldg(sv + e) + __ldg(tv + e);
      }
      if (fs.relu[k]) {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaxf(acc[e], 0.f);
      }
    }
    if (!valid) {
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    }
    uint4 o;
    uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) op[e] = pack2r(prog.fp16 != 0, acc[2 * e], acc[2 * e + 1]);
    *reinterpret_cast<uint4*>(prog.out_plane + row * prog.C + c0) = o;
    if (prog.out2_plane) {
#pragma unroll
      for (int e = 0; e < 4; ++e) op[e] = relu2r(prog.fp16 != 0, op[e]);  // relu commutes with the rounding
      *reinterpret_cast<uint4*>(prog.out2_plane + row * prog.C + c0) = o;
    }
  }
}

template <int NS>
void launch_fold_plane_t(const PwProgram& prog, const FoldSteps& fs, const PlaneGeom& geo, cudaStream_t s) {
  const int64_t total = geo.Nalloc * (prog.C / 8);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 32));
  pw_fold_plane_kernel<NS><<<blocks, 256, 0, s>>>(prog, fs, geo);
  CNRX_CUDA(cudaGetLastError());
}

bool launch_fold_plane(const PwProgram& prog, const FoldSteps& fs, int ns, const PlaneGeom& geo, cudaStream_t s) {
  if (prog.C % 8 != 0) return false;
  switch (ns) {
    case 1: launch_fold_plane_t<1>(prog, fs, geo, s); return true;
    case 2: launch_fold_plane_t<2>(prog, fs, geo, s); return true;
    case 3: launch_fold_plane_t<3>(prog, fs, geo, s); return true;
    case 4: launch_fold_plane_t<4>(prog, fs, geo, s); return true;
    default: return false;
  }
}

}  // namespace

bool pw_as_fold(const PwProgram& prog, int* nsteps, int* ops, int* affs, int* relus) {
  int ns = 0;
  for (int n = 0; n < prog.n_ins; ++n) {
    const PwIns& in = prog.ins[n];
    if (in.op == PW_LOAD || in.op == PW_MUL || in.op == PW_ADD) {
      if ((in.op == PW_LOAD) != (ns == 0) || in.k != ns || ns >= kPwMaxPlanes) return false;
      ops[ns] = in.op;
      affs[ns] = -1;
      relus[ns] = 0;
      ++ns;
    } else if (ns == 0) {
      return false;
    } else if (in.op == PW_AFF) {
      if (affs[ns - 1] >= 0 || relus[ns - 1]) return false;
      affs[ns - 1] = in.k;
    } else if (in.op == PW_RELU) {
      relus[ns - 1] = 1;
    }
  }
  *nsteps = ns;
  return ns > 0;
}

template <int HEAD, int LPR, bool SPLIT = false, int NPMAX = kPwMaxPlanes>
static void launch_rows(const PwProgram& prog, const PlaneGeom& geo, cudaStream_t s) {
  int n_aff = 0;
  for (int n = 0; n < prog.n_ins; ++n)
    if (prog.ins[n].op == PW_AFF) n_aff = std::max(n_aff, prog.ins[n].k + 1);
  const size_t smem = sizeof(float) * ((HEAD ? prog.C * prog.head_bits + ((prog.head_bits + 3) & ~3) : 0) +
                                       2 * n_aff * prog.C);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (geo.Nalloc + (32 / LPR) - 1) / (32 / LPR);
  const int64_t want = (groups + 15) / 16;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(want, static_cast<int64_t>(sms) * 8));
  pw_rows_kernel<HEAD, LPR, SPLIT, NPMAX><<<blocks, 256, smem, s>>>(prog, geo);
  CNRX_CUDA(cudaGetLastError());
}

namespace {
// one thread per 16-byte (8-channel) chunk of an output row half
__global__ void __launch_bounds__(256) concat_planes_kernel(const uint4* __restrict__ a, int ca8, const uint4* __restrict__ b,
                                                            int cb8, uint4* __restrict__ out, int halves, int64_t n) {
  const int c8 = ca8 + cb8;  // output chunks per half row
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / (halves * c8);
    const int r = static_cast<int>(i - row * halves * c8);
    const int h = r / c8, k = r - h * c8;  // half (hi / lo), chunk within the half
    out[i] = k < ca8 ? a[(row * halves + h) * ca8 + k] : b[(row * halves + h) * cb8 + (k - ca8)];
  }
}
}  // namespace

namespace {
// one thread per (row, 8-channel chunk)
__global__ void __launch_bounds__(256) dwconv_plane_kernel(const __nv_bfloat16* __restrict__ in, __nv_bfloat16* __restrict__ out,
                                                           const float* __restrict__ w, const float* __restrict__ bias, int C,
                                                           int kh, int kw, int dil, bool h16, bool split, PlaneGeom geo) {
  const int c8 = C / 8;
  const int64_t n = geo.Nalloc * c8;
  const int64_t rs = split ? 2 * C : C;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / c8;
    const int c0 = static_cast<int>(i - row * c8) * 8;
    float acc[8];
    const bool valid = geo.valid(row);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = valid && bias ? bias[c0 + e] : 0.f;
    if (valid) {
      for (int dt = 0; dt < kh; ++dt)
        for (int df = 0; df < kw; ++df) {
          const int64_t r2 = row + (dt - kh / 2) + static_cast<int64_t>(df - kw / 2) * dil * geo.T1;
          if (r2 < 0 || r2 >= geo.Nalloc) continue;  // zero rows (out-of-grid taps) contribute nothing
          float v[8];
          load8(in + r2 * rs + c0, v, h16);
          if (split) {
            float l[8];
            load8(in + r2 * rs + C + c0, l, h16);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] += l[e];
          }
          const float* wt = w + (dt * kw + df) * C + c0;
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], __fmul_rn(v[e], wt[e]));
        }
    }
    if (split) {
      store8_split(out + row * rs + c0, C, acc, h16);
    } else {
      uint4 o;
      uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) op[e] = pack2r(h16, acc[2 * e], acc[2 * e + 1]);
      *reinterpret_cast<uint4*>(out + row * C + c0) = o;
    }
  }
}
}  // namespace

const char* launch_dwconv_plane(const __nv_bfloat16* in, __nv_bfloat16* out, const float* w, const float* bias, int C,
                                int kh, int kw, int dil, bool h16, bool split, const PlaneGeom& geo, cudaStream_t s) {
  const int64_t n = geo.Nalloc * (C / 8);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  dwconv_plane_kernel<<<blocks, 256, 0, s>>>(in, out, w, bias, C, kh, kw, dil, h16, split, geo);
  CNRX_CUDA(cudaGetLastError());
  return split ? "dwconv_plane_kernel<x3>" : "dwconv_plane_kernel";
}

const char* launch_concat_planes(const __nv_bfloat16* a, int ca, const __nv_bfloat16* b, int cb, __nv_bfloat16* out,
                                 bool split, const PlaneGeom& geo, cudaStream_t s) {
  require(ca % 8 == 0 && cb % 8 == 0, "internal: concat channel counts must be multiples of 8");
  const int halves = split ? 2 : 1;
  const int64_t n = geo.Nalloc * halves * ((ca + cb) / 8);
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  concat_planes_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const uint4*>(a), ca / 8, reinterpret_cast<const uint4*>(b),
                                              cb / 8, reinterpret_cast<uint4*>(out), halves, n);
  CNRX_CUDA(cudaGetLastError());
  return split ? "concat_planes_kernel<x3>" : "concat_planes_kernel";
}

const char* launch_pw_program(const PwProgram& prog, const PlaneGeom& geo, cudaStream_t s) {
  if (prog.head_bits > 0) require(prog.head_bits <= kPwMaxBits, "head with more than 16 outputs");
  require(prog.out2_plane == nullptr || prog.head_bits == 0, "second output needs a plane program");
  const bool head = prog.head_bits > 0;
  if (prog.ln) {  // layer-norm program (plane output)
    require(!head && prog.C <= kLnMaxC && !prog.out2_plane, "internal: layer-norm program shape");
    pw_ln_kernel<<<static_cast<unsigned>((geo.Nalloc + 127) / 128), 128, 0, s>>>(prog, geo);
    CNRX_CUDA(cudaGetLastError());
    return prog.split ? "pw_ln_kernel<x3>" : "pw_ln_kernel";
  }
  if (prog.split && head) {  // split planes: the TMA-streamed head kernel reads hi + lo tiles when it fits
    FoldSteps fs{};
    int ns = 0;
    if (pw_as_fold(prog, &ns, fs.op, fs.aff, fs.relu) && prog.n_planes_used == ns) {
      const char* name = launch_head_tma(prog, ns, fs.op, fs.aff, fs.relu, geo, s);
      if (name) return "head_tma_kernel<x3>";
    }
  }
  if (prog.split && !prog.out2_plane && prog.n_planes_used <= 4 && (prog.C == 16 || prog.C == 32 || prog.C == 64) &&
      !head) {
    // split planes, coalesced: a row's lanes read their slices of both halves (<= 4 operand planes: the
    // register arrays are sized for them)
    switch (prog.C) {
      case 16: head ? launch_rows<1, 2, true, 4>(prog, geo, s) : launch_rows<0, 2, true, 4>(prog, geo, s); break;
      case 32: head ? launch_rows<1, 4, true, 4>(prog, geo, s) : launch_rows<0, 4, true, 4>(prog, geo, s); break;
      default: head ? launch_rows<1, 8, true, 4>(prog, geo, s) : launch_rows<0, 8, true, 4>(prog, geo, s); break;
    }
    return head ? "pw_rows_kernel<head,x3>" : "pw_rows_kernel<plane,x3>";
  }
  if (prog.split) {  // other widths / a second output: the generic interpreter (one thread per row)
    const int threads = 256;
    const unsigned blocks = static_cast<unsigned>((geo.Nalloc + threads - 1) / threads);
    if (head) {
      const size_t smem = sizeof(float) * (static_cast<size_t>(prog.C) * prog.head_bits + prog.head_bits);
      pw_program_kernel<1><<<blocks, threads, smem, s>>>(prog, geo);
    } else {
      pw_program_kernel<0><<<blocks, threads, 0, s>>>(prog, geo);
    }
    CNRX_CUDA(cudaGetLastError());
    return head ? "pw_program_kernel<head,x3>" : "pw_program_kernel<plane,x3>";
  }
  {
    FoldSteps fs{};
    int ns = 0;
    if (pw_as_fold(prog, &ns, fs.op, fs.aff, fs.relu) && prog.n_planes_used == ns) {
      // the TMA-streamed head kernel (tensor-core GEMV over bf16 z when the plan asks for it, else fp32)
      if (head) {
        const char* name = launch_head_tma(prog, ns, fs.op, fs.aff, fs.relu, geo, s);
        if (name) return name;
      }
      if (!head && launch_fold_plane(prog, fs, ns, geo, s)) return "pw_fold_plane_kernel";
      const bool ok = launch_fold_any(prog, fs, ns, geo, s);
      if (ok) return head ? "pw_fold_kernel<head>" : "pw_fold_kernel<plane>";
    }
  }
  require(prog.out2_plane == nullptr, "internal: a second pointwise output needs a fold program");
  switch (prog.C) {
    case 16: head ? launch_rows<1, 2>(prog, geo, s) : launch_rows<0, 2>(prog, geo, s); break;
    case 32: head ? launch_rows<1, 4>(prog, geo, s) : launch_rows<0, 4>(prog, geo, s); break;
    case 64: head ? launch_rows<1, 8>(prog, geo, s) : launch_rows<0, 8>(prog, geo, s); break;
    case 128: head ? launch_rows<1, 16>(prog, geo, s) : launch_rows<0, 16>(prog, geo, s); break;
    default: {
      const int threads = 256;
      const unsigned blocks = static_cast<unsigned>((geo.Nalloc + threads - 1) / threads);
      if (head) {
        const size_t smem = sizeof(float) * (static_cast<size_t>(prog.C) * prog.head_bits + prog.head_bits);
        pw_program_kernel<1><<<blocks, threads, smem, s>>>(prog, geo);
      } else {
        pw_program_kernel<0><<<blocks, threads, 0, s>>>(prog, geo);
      }
      CNRX_CUDA(cudaGetLastError());
      return head ? "pw_program_kernel<head>" : "pw_program_kernel<plane>";
    }
  }
  return head ? "pw_rows_kernel<head>" : "pw_rows_kernel<plane>";
}

}  // namespace cnrx
