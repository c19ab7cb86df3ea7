// featurize.cu — received grid -> network input features (HBM-bound gather, one pass).
//
// Replaces the reference's featurizer, format_nn_input (listed at
// proj/core/CMakeLists.txt:7 but missing from the snapshot) together with the LS pilot estimate and
// its interpolation (classic.cpp, also missing), adapted to BASELINE's feature set:
// per receive antenna a, channels 6a..6a+5 = [Re y, Im y, Re x_p, Im x_p, Re h_ls, Im h_ls], where x_p
// is the pilot grid (0 off-pilot) and h_ls the LS estimate y/x_p at pilot REs, interpolated linearly
// along F inside each pilot symbol (nearest beyond the edge pilots) and linearly along T between pilot
// symbols (nearest outside).  Restated in oracle/oracle.c:orc_featurize.
//
// One thread per (slot, frequency column): it reads the column's pilot-symbol LS values once, then
// walks the T symbols.  Warp lanes are consecutive subcarriers, so y reads are coalesced
// ([B,T,F,N] complex, antenna fastest); plane writes are whole 32 B sectors per row.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "kernels.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kMaxN = 8;

struct Cplx {
  float re, im;
};
__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// Computes the 6N features of (b, t, f) given per-pilot-symbol LS values hs[j][a] at column f.
// NT / NS > 0: antenna and pilot-symbol counts known at compile time, so the per-column LS values and
// the feature vector live in registers (the generic form indexes them at run time: an 816-byte stack
// frame in local memory).
template <int OUT_PLANE, int NT = 0, int NS = 0>
__global__ void featurize_kernel(const float2* __restrict__ y, PlaneGeom geo, int N_rt, PilotTablesDev pt,
                                 float* __restrict__ feat_ref, __nv_bfloat16* __restrict__ plane, int cpad, bool h16) {
  const int N = NT > 0 ? NT : N_rt;
  constexpr int kN = NT > 0 ? NT : kMaxN;
  constexpr int kS = NS > 0 ? NS : kMaxPilotSyms;
  const int64_t cols_per_slot = geo.F + geo.npad;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n_cols = static_cast<int64_t>(geo.B) * cols_per_slot;
  const int T = geo.T, F = geo.F;
  if (OUT_PLANE) {
    // tail: zero rows [B*P, Nalloc) handled by the first threads of an extra range
    const int64_t tail0 = static_cast<int64_t>(geo.B) * geo.P;
    const int64_t ntail = geo.Nalloc - tail0;
    if (idx >= n_cols) {
      const int64_t r = idx - n_cols;
      if (r < ntail) {
        uint4* dst = reinterpret_cast<uint4*>(plane + (tail0 + r) * cpad);
        for (int i = 0; i < cpad / 8; ++i) dst[i] = make_uint4(0, 0, 0, 0);
      }
      return;
    }
  } else if (idx >= static_cast<int64_t>(geo.B) * F) {
    return;
  }
  int b, c;
  if (OUT_PLANE) {
    b = static_cast<int>(idx / cols_per_slot);
    c = static_cast<int>(idx - static_cast<int64_t>(b) * cols_per_slot);
  } else {
    b = static_cast<int>(idx / F);
    c = static_cast<int>(idx - static_cast<int64_t>(b) * F) + geo.npad;
  }
  const int f = c - geo.npad;
  if (OUT_PLANE && f < 0) {  // zero padding column
    for (int t = 0; t < geo.T1; ++t) {
      uint4* dst = reinterpret_cast<uint4*>(plane + geo.row_of(b, t, f) * cpad);
      for (int i = 0; i < cpad / 8; ++i) dst[i] = make_uint4(0, 0, 0, 0);
    }
    return;
  }
  // LS estimate at every pilot symbol, interpolated along F to this column.
  Cplx hs[kS][kN];
  const int n_sym = NS > 0 ? NS : pt.n_sym;
#pragma unroll
  for (int j = 0; j < kS; ++j) {
    if (j >= n_sym) break;
    const int ts = pt.sym[j];
    const int flo = pt.flo[j * F + f], fhi = pt.fhi[j * F + f];
    const float w = pt.wf[j * F + f];
    const Cplx ilo = {pt.inv_x[2 * (ts * F + flo)], pt.inv_x[2 * (ts * F + flo) + 1]};
    const Cplx ihi = {pt.inv_x[2 * (ts * F + fhi)], pt.inv_x[2 * (ts * F + fhi) + 1]};
#pragma unroll
    for (int a = 0; a < kN; ++a) {
      if (a >= N) break;
      const float2 ylo = y[((static_cast<int64_t>(b) * T + ts) * F + flo) * N + a];
      const float2 yhi = y[((static_cast<int64_t>(b) * T + ts) * F + fhi) * N + a];
      const Cplx llo = cmul({ylo.x, ylo.y}, ilo), lhi = cmul({yhi.x, yhi.y}, ihi);
      hs[j][a] = {(1.f - w) * llo.re + w * lhi.re, (1.f - w) * llo.im + w * lhi.im};
    }
  }
  for (int t = 0; t < (OUT_PLANE ? geo.T1 : T); ++t) {
    float v[6 * kN];
    const int C = 6 * N;
    if (t < T) {
      const int j0 = pt.jlo[t], j1 = pt.jhi[t];
      const float wt = pt.wt[t];
      const float xr = pt.x[2 * (t * F + f)], xi = pt.x[2 * (t * F + f) + 1];
#pragma unroll
      for (int a = 0; a < kN; ++a) {
        if (a >= N) break;
        // hs[j0][a], hs[j1][a] by static indices (selects), so hs stays in registers
        Cplx h0 = hs[0][a], h1 = hs[0][a];
#pragma unroll
        for (int j = 1; j < kS; ++j) {
          if (j == j0) h0 = hs[j][a];
          if (j == j1) h1 = hs[j][a];
        }
        const float2 yv = y[((static_cast<int64_t>(b) * T + t) * F + f) * N + a];
        v[6 * a + 0] = yv.x;
        v[6 * a + 1] = yv.y;
        v[6 * a + 2] = xr;
        v[6 * a + 3] = xi;
        v[6 * a + 4] = (1.f - wt) * h0.re + wt * h1.re;
        v[6 * a + 5] = (1.f - wt) * h0.im + wt * h1.im;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 6 * kN; ++i) v[i] = 0.f;
    }
    if (OUT_PLANE && cpad == 16) {  // one 32-byte row: a single 256-bit store
      u32x8 o;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = 2 * i;
        o.v[i] = pack2r(h16, k < C ? v[k] : 0.f, k + 1 < C ? v[k + 1] : 0.f);
      }
      stg256(plane + geo.row_of(b, t, f) * cpad, o);
    } else if (OUT_PLANE) {
      __nv_bfloat16* dst = plane + geo.row_of(b, t, f) * cpad;
#pragma unroll
      for (int i0 = 0; i0 < (6 * kN + 15) / 16 * 16; i0 += 8) {
        if (i0 >= cpad) break;
        uint4 o;
        uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = i0 + 2 * i;
          op[i] = pack2r(h16, k < C ? v[k] : 0.f, k + 1 < C ? v[k + 1] : 0.f);
        }
        *reinterpret_cast<uint4*>(dst + i0) = o;
      }
    } else {
      float* dst = feat_ref + ((static_cast<int64_t>(b) * T + t) * F + f) * C;
      for (int i = 0; i < C; ++i) dst[i] = v[i];
    }
  }
}

// Reference-layout fp32 features [B,T,F,C] -> bf16 / fp16 plane [Nalloc][cpad] (used by cnrx_forward
// when the caller supplies features rather than the received grid).
__global__ void pack_plane_kernel(const float* __restrict__ x, PlaneGeom geo, int C, __nv_bfloat16* __restrict__ plane,
                                  int cpad, bool h16, bool split) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= geo.Nalloc) return;
  // split planes (CNRX_*X3 plans): row = [hi cpad | lo cpad], hi = round16(v), lo = round16(v - hi)
  __nv_bfloat16* dst = plane + row * (split ? 2 * cpad : cpad);
  const bool valid = geo.valid(row);
  const float* src = nullptr;
  if (valid) {
    int b, t, f;
    geo.coords(row, b, t, f);
    src = x + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * C;
  }
  for (int i0 = 0; i0 < cpad; i0 += 8) {
    uint4 o, ol;
    uint32_t* op = reinterpret_cast<uint32_t*>(&o);
    uint32_t* opl = reinterpret_cast<uint32_t*>(&ol);
    for (int i = 0; i < 4; ++i) {
      const int k = i0 + 2 * i;
      const float a = (valid && k < C) ? src[k] : 0.f;
      const float c = (valid && k + 1 < C) ? src[k + 1] : 0.f;
      op[i] = pack2r(h16, a, c);
      const float2 hf = unpack2r(h16, op[i]);
      opl[i] = pack2r(h16, a - hf.x, c - hf.y);
    }
    *reinterpret_cast<uint4*>(dst + i0) = o;
    if (split) *reinterpret_cast<uint4*>(dst + cpad + i0) = ol;
  }
}

// Features of plane row `row` (valid rows only): receive mode restates featurize_kernel per row.
template <int CIN>
__device__ __forceinline__ void row_features(const StemLaunch& L, const PlaneGeom& geo, int b, int t, int f,
                                             float (&v)[CIN]) {
  if (L.mode == 0) {
    const float* src = L.x + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * CIN;
#pragma unroll
    for (int i = 0; i < CIN; ++i) v[i] = src[i];
    return;
  }
  const PilotTablesDev& pt = L.pt;
  constexpr int N = CIN / 6;
  const int T = geo.T, F = geo.F;
  const float2* y = reinterpret_cast<const float2*>(L.y);
  const int j0 = pt.jlo[t], j1 = pt.jhi[t];
  const float wt = pt.wt[t];
  const float xr = pt.x[2 * (t * F + f)], xi = pt.x[2 * (t * F + f) + 1];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    Cplx h[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int jj = q == 0 ? j0 : j1;
      const int ts = pt.sym[jj];
      const int flo = pt.flo[jj * F + f], fhi = pt.fhi[jj * F + f];
      const float w = pt.wf[jj * F + f];
      const Cplx ilo = {pt.inv_x[2 * (ts * F + flo)], pt.inv_x[2 * (ts * F + flo) + 1]};
      const Cplx ihi = {pt.inv_x[2 * (ts * F + fhi)], pt.inv_x[2 * (ts * F + fhi) + 1]};
      const float2 ylo = y[((static_cast<int64_t>(b) * T + ts) * F + flo) * N + a];
      const float2 yhi = y[((static_cast<int64_t>(b) * T + ts) * F + fhi) * N + a];
      const Cplx llo = cmul({ylo.x, ylo.y}, ilo), lhi = cmul({yhi.x, yhi.y}, ihi);
      h[q] = {(1.f - w) * llo.re + w * lhi.re, (1.f - w) * llo.im + w * lhi.im};
    }
    const float2 yv = y[((static_cast<int64_t>(b) * T + t) * F + f) * N + a];
    v[6 * a + 0] = yv.x;
    v[6 * a + 1] = yv.y;
    v[6 * a + 2] = xr;
    v[6 * a + 3] = xi;
    v[6 * a + 4] = (1.f - wt) * h[0].re + wt * h[1].re;
    v[6 * a + 5] = (1.f - wt) * h[0].im + wt * h[1].im;
  }
}

// Fused input stage.  grid.y = stem op; eight lanes share a plane row and lane g owns output
// channels [8g, 8g+8) of the op, keeping its 8 x CIN weight slice in registers for the whole kernel,
// so a row is written as one contiguous 128-byte line (a warp instruction stores 4 full rows).
// The N antennas' 6 features are computed by the row's first N lanes and broadcast with shuffles.
template <int CIN>
__global__ void __launch_bounds__(256) stem_kernel(const __grid_constant__ StemLaunch L, PlaneGeom geo) {
  constexpr int N = CIN / 6;
  const StemOp& op = L.op[blockIdx.y];
  const int cout = op.cout;
  const int lane = threadIdx.x & 31;
  const int g = lane & 7;         // 16-byte chunk of the row this lane writes
  const int rsub = lane >> 3;     // row within the warp's 4-row group
  const int base_lane = lane & ~7;
  const int c0 = g * 8;
  const bool active = c0 < cout;
  float wr[CIN][8], bias[8], s2[8], t2[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = active ? c0 + k : 0;
#pragma unroll
    for (int i = 0; i < CIN; ++i) wr[i][k] = op.w[i * cout + c];
    bias[k] = op.bias[c];
    s2[k] = op.s2 ? op.s2[c] : 1.f;
    t2[k] = op.t2 ? op.t2[c] : 0.f;
  }
  const int64_t groups = (geo.Nalloc + 3) / 4;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t wg = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); wg < groups;
       wg += wstride) {
    const int64_t row = wg * 4 + rsub;
    const bool in_range = row < geo.Nalloc;
    const bool valid = in_range && geo.valid(row);
    float mine[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) mine[k] = 0.f;
    if (valid && g < N) {
      int b, t, f;
      geo.coords(row, b, t, f);
      if (L.mode == 0) {
        const float* src = L.x + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * CIN + 6 * g;
#pragma unroll
        for (int k = 0; k < 6; ++k) mine[k] = src[k];
      } else {
        const PilotTablesDev& pt = L.pt;
        const int T = geo.T, F = geo.F;
        const float2* y = reinterpret_cast<const float2*>(L.y);
        const int j0 = pt.jlo[t], j1 = pt.jhi[t];
        const float wt = pt.wt[t];
        Cplx h[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int jj = q == 0 ? j0 : j1;
          const int ts = pt.sym[jj];
          const int flo = pt.flo[jj * F + f], fhi = pt.fhi[jj * F + f];
          const float w = pt.wf[jj * F + f];
          const Cplx ilo = {pt.inv_x[2 * (ts * F + flo)], pt.inv_x[2 * (ts * F + flo) + 1]};
          const Cplx ihi = {pt.inv_x[2 * (ts * F + fhi)], pt.inv_x[2 * (ts * F + fhi) + 1]};
          const float2 ylo = y[((static_cast<int64_t>(b) * T + ts) * F + flo) * N + g];
          const float2 yhi = y[((static_cast<int64_t>(b) * T + ts) * F + fhi) * N + g];
          const Cplx llo = cmul({ylo.x, ylo.y}, ilo), lhi = cmul({yhi.x, yhi.y}, ihi);
          h[q] = {(1.f - w) * llo.re + w * lhi.re, (1.f - w) * llo.im + w * lhi.im};
        }
        const float2 yv = y[((static_cast<int64_t>(b) * T + t) * F + f) * N + g];
        mine[0] = yv.x;
        mine[1] = yv.y;
        mine[2] = pt.x[2 * (t * F + f)];
        mine[3] = pt.x[2 * (t * F + f) + 1];
        mine[4] = (1.f - wt) * h[0].re + wt * h[1].re;
        mine[5] = (1.f - wt) * h[0].im + wt * h[1].im;
      }
    }
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = bias[k];
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int k6 = 0; k6 < 6; ++k6) {
        const float xi = __shfl_sync(0xffffffffu, mine[k6], base_lane + a);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = fmaf(xi, wr[6 * a + k6][k], acc[k]);
      }
    if (!active || !in_range) continue;
    uint4 o1, o2;
    uint32_t* p1 = reinterpret_cast<uint32_t*>(&o1);
    uint32_t* p2 = reinterpret_cast<uint32_t*>(&o2);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float a0 = acc[2 * k], a1 = acc[2 * k + 1];
      if (op.relu) {
        a0 = fmaxf(a0, 0.f);
        a1 = fmaxf(a1, 0.f);
      }
      if (!valid) a0 = a1 = 0.f;
      p1[k] = pack2r(L.fp16 != 0, a0, a1);
      const float u0 = valid ? fmaxf(a0 * s2[2 * k] + t2[2 * k], 0.f) : 0.f;
      const float u1 = valid ? fmaxf(a1 * s2[2 * k + 1] + t2[2 * k + 1], 0.f) : 0.f;
      p2[k] = pack2r(L.fp16 != 0, u0, u1);
    }
    *reinterpret_cast<uint4*>(op.out + row * cout + c0) = o1;
    if (op.out2) *reinterpret_cast<uint4*>(op.out2 + row * cout + c0) = o2;
  }
}

// Small batches: one thread per plane row (slot, column, symbol) instead of per column, so a single
// slot still spreads over the GPU; each thread recomputes its column's LS values at the two pilot
// symbols it interpolates between (a handful of L1/L2-resident loads).
__global__ void featurize_row_kernel(const float2* __restrict__ y, PlaneGeom geo, int N, PilotTablesDev pt,
                                     __nv_bfloat16* __restrict__ plane, int cpad, bool h16) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= geo.Nalloc) return;
  float v[6 * kMaxN];
  const int C = 6 * N;
  for (int i = 0; i < C; ++i) v[i] = 0.f;
  if (geo.valid(row)) {
    int b, t, f;
    geo.coords(row, b, t, f);
    const int T = geo.T, F = geo.F;
    const int j0 = pt.jlo[t], j1 = pt.jhi[t];
    const float wt = pt.wt[t];
    Cplx hs[2][kMaxN];
    for (int jj = 0; jj < 2; ++jj) {
      const int j = jj == 0 ? j0 : j1;
      const int ts = pt.sym[j];
      const int flo = pt.flo[j * F + f], fhi = pt.fhi[j * F + f];
      const float w = pt.wf[j * F + f];
      const Cplx ilo = {pt.inv_x[2 * (ts * F + flo)], pt.inv_x[2 * (ts * F + flo) + 1]};
      const Cplx ihi = {pt.inv_x[2 * (ts * F + fhi)], pt.inv_x[2 * (ts * F + fhi) + 1]};
      for (int a = 0; a < N; ++a) {
        const float2 ylo = y[((static_cast<int64_t>(b) * T + ts) * F + flo) * N + a];
        const float2 yhi = y[((static_cast<int64_t>(b) * T + ts) * F + fhi) * N + a];
        const Cplx llo = cmul({ylo.x, ylo.y}, ilo), lhi = cmul({yhi.x, yhi.y}, ihi);
        hs[jj][a] = {(1.f - w) * llo.re + w * lhi.re, (1.f - w) * llo.im + w * lhi.im};
      }
    }
    const float xr = pt.x[2 * (t * F + f)], xi = pt.x[2 * (t * F + f) + 1];
    for (int a = 0; a < N; ++a) {
      const float2 yv = y[((static_cast<int64_t>(b) * T + t) * F + f) * N + a];
      v[6 * a + 0] = yv.x;
      v[6 * a + 1] = yv.y;
      v[6 * a + 2] = xr;
      v[6 * a + 3] = xi;
      v[6 * a + 4] = (1.f - wt) * hs[0][a].re + wt * hs[1][a].re;
      v[6 * a + 5] = (1.f - wt) * hs[0][a].im + wt * hs[1][a].im;
    }
  }
  __nv_bfloat16* dst = plane + row * cpad;
  for (int i0 = 0; i0 < cpad; i0 += 8) {
    uint4 o;
    uint32_t* op = reinterpret_cast<uint32_t*>(&o);
    for (int i = 0; i < 4; ++i) {
      const int k = i0 + 2 * i;
      op[i] = pack2r(h16, k < C ? v[k] : 0.f, k + 1 < C ? v[k + 1] : 0.f);
    }
    *reinterpret_cast<uint4*>(dst + i0) = o;
  }
}

}  // namespace

bool stem_supported_cin(int cin) { return cin == 6 || cin == 12 || cin == 24 || cin == 48; }

const char* launch_stem(const StemLaunch& L, const PlaneGeom& geo, cudaStream_t s) {
  require(L.cin <= kStemMaxIn && L.nops >= 1 && L.nops <= kStemMaxOps, "stem launch out of range");
  for (int i = 0; i < L.nops; ++i)
    require(L.op[i].cout <= 64 && L.op[i].cout % 8 == 0, "stem kernel writes <= 64 channels per op");
  const size_t smem = 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (geo.Nalloc + 3) / 4;
  const dim3 blocks(static_cast<unsigned>(std::min<int64_t>((groups + 7) / 8, static_cast<int64_t>(sms) * 4)),
                    static_cast<unsigned>(L.nops));
  switch (L.cin) {
    case 6: stem_kernel<6><<<blocks, 256, smem, s>>>(L, geo); break;
    case 12: stem_kernel<12><<<blocks, 256, smem, s>>>(L, geo); break;
    case 24: stem_kernel<24><<<blocks, 256, smem, s>>>(L, geo); break;
    case 48: stem_kernel<48><<<blocks, 256, smem, s>>>(L, geo); break;
    default: throw Error(3, "stem kernel supports 6/12/24/48 input channels");
  }
  CNRX_CUDA(cudaGetLastError());
  return L.mode == 1 ? "stem_kernel<featurize>" : "stem_kernel<features>";
}

const char* launch_featurize_plane(const float* y, const PlaneGeom& geo, int N, const PilotTablesDev& pt,
                                   __nv_bfloat16* plane, int cpad, bool fp16, cudaStream_t s) {
  require(N <= kMaxN, "featurize supports at most 8 receive antennas");
  const int64_t n = static_cast<int64_t>(geo.B) * (geo.F + geo.npad) + (geo.Nalloc - static_cast<int64_t>(geo.B) * geo.P);
  const int threads = 128;
  if (n < 148 * 128 && pt.n_sym >= 1) {  // too few columns to fill the GPU: one thread per row
    featurize_row_kernel<<<static_cast<unsigned>((geo.Nalloc + threads - 1) / threads), threads, 0, s>>>(
        reinterpret_cast<const float2*>(y), geo, N, pt, plane, cpad, fp16);
    CNRX_CUDA(cudaGetLastError());
    return "featurize_row_kernel";
  }
  const unsigned blocks = static_cast<unsigned>((n + threads - 1) / threads);
  const float2* y2 = reinterpret_cast<const float2*>(y);
  if (pt.n_sym == 2 && N == 2)  // the BASELINE DM-RS layout (2 pilot symbols) with 2 / 1 / 4 antennas
    featurize_kernel<1, 2, 2><<<blocks, threads, 0, s>>>(y2, geo, N, pt, nullptr, plane, cpad, fp16);
  else if (pt.n_sym == 2 && N == 1)
    featurize_kernel<1, 1, 2><<<blocks, threads, 0, s>>>(y2, geo, N, pt, nullptr, plane, cpad, fp16);
  else if (pt.n_sym == 2 && N == 4)
    featurize_kernel<1, 4, 2><<<blocks, threads, 0, s>>>(y2, geo, N, pt, nullptr, plane, cpad, fp16);
  else
    featurize_kernel<1><<<blocks, threads, 0, s>>>(y2, geo, N, pt, nullptr, plane, cpad, fp16);
  CNRX_CUDA(cudaGetLastError());
  return "featurize_kernel<plane>";
}

const char* launch_featurize_ref(const float* y, const PlaneGeom& geo, int N, const PilotTablesDev& pt, float* feat,
                                 cudaStream_t s) {
  require(N <= kMaxN, "featurize supports at most 8 receive antennas");
  const int64_t n = static_cast<int64_t>(geo.B) * geo.F;
  const int threads = 128;
  featurize_kernel<0><<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, s>>>(
      reinterpret_cast<const float2*>(y), geo, N, pt, feat, nullptr, 0, false);
  CNRX_CUDA(cudaGetLastError());
  return "featurize_kernel<ref>";
}

namespace {
__global__ void plane_rows_to_ref_kernel(const uint16_t* __restrict__ plane, PlaneGeom geo, int cpad,
                                         uint16_t* __restrict__ out) {
  const int64_t n = static_cast<int64_t>(geo.B) * geo.T * geo.F * cpad;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = i % cpad, r = i / cpad;
    const int f = static_cast<int>(r % geo.F), t = static_cast<int>((r / geo.F) % geo.T);
    const int b = static_cast<int>(r / (static_cast<int64_t>(geo.F) * geo.T));
    out[i] = plane[geo.row_of(b, t, f) * cpad + c];
  }
}
}  // namespace

const char* launch_plane_rows_to_ref(const __nv_bfloat16* plane, const PlaneGeom& geo, int cpad, uint16_t* out,
                                     cudaStream_t s) {
  plane_rows_to_ref_kernel<<<1024, 256, 0, s>>>(reinterpret_cast<const uint16_t*>(plane), geo, cpad, out);
  CNRX_CUDA(cudaGetLastError());
  return "plane_rows_to_ref_kernel";
}

const char* launch_pack_plane(const float* x, const PlaneGeom& geo, int C, __nv_bfloat16* plane, int cpad, bool fp16,
                              cudaStream_t s, bool split) {
  const int threads = 256;
  pack_plane_kernel<<<static_cast<unsigned>((geo.Nalloc + threads - 1) / threads), threads, 0, s>>>(x, geo, C, plane,
                                                                                                   cpad, fp16, split);
  CNRX_CUDA(cudaGetLastError());
  if (split) return "pack_plane_kernel<x3>";
  return "pack_plane_kernel";
}

}  // namespace cnrx
