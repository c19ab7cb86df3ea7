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

#include "common.h"
#include "kernels.h"

namespace cnrx {

namespace {

constexpr int kMaxN = 8;

struct Cplx {
  float re, im;
};
__device__ __forceinline__ Cplx cmul(Cplx a, Cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// Computes the 6N features of (b, t, f) given per-pilot-symbol LS values hs[j][a] at column f.
template <int OUT_PLANE>
__global__ void featurize_kernel(const float2* __restrict__ y, PlaneGeom geo, int N, PilotTablesDev pt,
                                 float* __restrict__ feat_ref, __nv_bfloat16* __restrict__ plane, int cpad) {
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
  Cplx hs[kMaxPilotSyms][kMaxN];
  for (int j = 0; j < pt.n_sym; ++j) {
    const int ts = pt.sym[j];
    const int flo = pt.flo[j * F + f], fhi = pt.fhi[j * F + f];
    const float w = pt.wf[j * F + f];
    const Cplx ilo = {pt.inv_x[2 * (ts * F + flo)], pt.inv_x[2 * (ts * F + flo) + 1]};
    const Cplx ihi = {pt.inv_x[2 * (ts * F + fhi)], pt.inv_x[2 * (ts * F + fhi) + 1]};
    for (int a = 0; a < N; ++a) {
      const float2 ylo = y[((static_cast<int64_t>(b) * T + ts) * F + flo) * N + a];
      const float2 yhi = y[((static_cast<int64_t>(b) * T + ts) * F + fhi) * N + a];
      const Cplx llo = cmul({ylo.x, ylo.y}, ilo), lhi = cmul({yhi.x, yhi.y}, ihi);
      hs[j][a] = {(1.f - w) * llo.re + w * lhi.re, (1.f - w) * llo.im + w * lhi.im};
    }
  }
  for (int t = 0; t < (OUT_PLANE ? geo.T1 : T); ++t) {
    float v[6 * kMaxN];
    const int C = 6 * N;
    if (t < T) {
      const int j0 = pt.jlo[t], j1 = pt.jhi[t];
      const float wt = pt.wt[t];
      const float xr = pt.x[2 * (t * F + f)], xi = pt.x[2 * (t * F + f) + 1];
      for (int a = 0; a < N; ++a) {
        const float2 yv = y[((static_cast<int64_t>(b) * T + t) * F + f) * N + a];
        v[6 * a + 0] = yv.x;
        v[6 * a + 1] = yv.y;
        v[6 * a + 2] = xr;
        v[6 * a + 3] = xi;
        v[6 * a + 4] = (1.f - wt) * hs[j0][a].re + wt * hs[j1][a].re;
        v[6 * a + 5] = (1.f - wt) * hs[j0][a].im + wt * hs[j1][a].im;
      }
    } else {
      for (int i = 0; i < C; ++i) v[i] = 0.f;
    }
    if (OUT_PLANE) {
      __nv_bfloat16* dst = plane + geo.row_of(b, t, f) * cpad;
      for (int i0 = 0; i0 < cpad; i0 += 8) {
        uint4 o;
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&o);
        for (int i = 0; i < 4; ++i) {
          const int k = i0 + 2 * i;
          op[i] = __floats2bfloat162_rn(k < C ? v[k] : 0.f, k + 1 < C ? v[k + 1] : 0.f);
        }
        *reinterpret_cast<uint4*>(dst + i0) = o;
      }
    } else {
      float* dst = feat_ref + ((static_cast<int64_t>(b) * T + t) * F + f) * C;
      for (int i = 0; i < C; ++i) dst[i] = v[i];
    }
  }
}

// Reference-layout fp32 features [B,T,F,C] -> bf16 plane [Nalloc][cpad] (used by cnrx_forward when
// the caller supplies features rather than the received grid).
__global__ void pack_plane_kernel(const float* __restrict__ x, PlaneGeom geo, int C, __nv_bfloat16* __restrict__ plane,
                                  int cpad) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= geo.Nalloc) return;
  __nv_bfloat16* dst = plane + row * cpad;
  const bool valid = geo.valid(row);
  const float* src = nullptr;
  if (valid) {
    int b, t, f;
    geo.coords(row, b, t, f);
    src = x + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * C;
  }
  for (int i0 = 0; i0 < cpad; i0 += 8) {
    uint4 o;
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&o);
    for (int i = 0; i < 4; ++i) {
      const int k = i0 + 2 * i;
      const float a = (valid && k < C) ? src[k] : 0.f;
      const float c = (valid && k + 1 < C) ? src[k + 1] : 0.f;
      op[i] = __floats2bfloat162_rn(a, c);
    }
    *reinterpret_cast<uint4*>(dst + i0) = o;
  }
}

}  // namespace

const char* launch_featurize_plane(const float* y, const PlaneGeom& geo, int N, const PilotTablesDev& pt,
                                   __nv_bfloat16* plane, int cpad, cudaStream_t s) {
  require(N <= kMaxN, "featurize supports at most 8 receive antennas");
  const int64_t n = static_cast<int64_t>(geo.B) * (geo.F + geo.npad) + (geo.Nalloc - static_cast<int64_t>(geo.B) * geo.P);
  const int threads = 128;
  featurize_kernel<1><<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, s>>>(
      reinterpret_cast<const float2*>(y), geo, N, pt, nullptr, plane, cpad);
  CNRX_CUDA(cudaGetLastError());
  return "featurize_kernel<plane>";
}

const char* launch_featurize_ref(const float* y, const PlaneGeom& geo, int N, const PilotTablesDev& pt, float* feat,
                                 cudaStream_t s) {
  require(N <= kMaxN, "featurize supports at most 8 receive antennas");
  const int64_t n = static_cast<int64_t>(geo.B) * geo.F;
  const int threads = 128;
  featurize_kernel<0><<<static_cast<unsigned>((n + threads - 1) / threads), threads, 0, s>>>(
      reinterpret_cast<const float2*>(y), geo, N, pt, feat, nullptr, 0);
  CNRX_CUDA(cudaGetLastError());
  return "featurize_kernel<ref>";
}

const char* launch_pack_plane(const float* x, const PlaneGeom& geo, int C, __nv_bfloat16* plane, int cpad,
                              cudaStream_t s) {
  const int threads = 256;
  pack_plane_kernel<<<static_cast<unsigned>((geo.Nalloc + threads - 1) / threads), threads, 0, s>>>(x, geo, C, plane,
                                                                                                   cpad);
  CNRX_CUDA(cudaGetLastError());
  return "pack_plane_kernel";
}

}  // namespace cnrx
