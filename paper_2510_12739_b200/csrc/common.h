// common.h — definitions shared by the host runtime (api.cpp) and the kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <cstdlib>
#include <string>
#include <utility>

namespace cnrx {

// Error type carrying a C-ABI status code.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// ---------------------------------------------------------------------------------------------
// Plane layout.  A bf16 activation "plane" stores one graph value
// for a whole slot batch as rows of C channels.  Within a slot the grid is stored frequency-column
// by column with the T symbols of a column contiguous, followed by one zero row, and each slot is
// preceded by `npad` all-zero columns:
//
//     row(b, f, t) = b*P + (f + npad)*(T+1) + t,    P = (F + npad)*(T+1)
//
// plus npad trailing zero columns after the last slot.  With that padding a 3x3 "same" convolution
// (dilation d <= npad along F) is a 1-D stencil over rows with offsets (dt-1) + (df-1)*d*(T+1): every
// tap that falls outside the grid lands on a zero row, so the implicit GEMM needs no masking.
// Rows that are padding are kept at zero by every kernel that writes a plane.
// ---------------------------------------------------------------------------------------------
// Division by a runtime constant via multiply-high (valid for dividends < 2^31), as in CUTLASS's
// FastDivmod: 64-bit integer division costs ~100 instructions on the GPU.
struct FastDiv {
  uint32_t d, mul, shr;
  __host__ __device__ uint32_t div(uint32_t n) const {
#ifdef __CUDA_ARCH__
    return d == 1 ? n : (__umulhi(n, mul) >> shr);
#else
    return d == 1 ? n : static_cast<uint32_t>((static_cast<uint64_t>(n) * mul >> 32) >> shr);
#endif
  }
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d != 1) {
    int l = 0;
    while ((1u << l) < d) ++l;  // ceil(log2 d)
    const int p = 31 + l;
    f.mul = static_cast<uint32_t>(((1ull << p) + d - 1) / d);
    f.shr = static_cast<uint32_t>(p - 32);
  }
  return f;
}

struct PlaneGeom {
  int32_t B, T, F, npad;
  int32_t T1;       // T + 1 rows per frequency column
  int64_t P;        // rows per slot
  int64_t Npos;     // B*P + npad*T1
  int64_t Nalloc;   // Npos rounded up to the 128-row GEMM tile
  int64_t n_tiles;  // Nalloc / 128
  FastDiv divP, divT1;

  __host__ __device__ bool valid(int64_t row) const {
    if (row >= static_cast<int64_t>(B) * P) return false;
    const uint32_t n = static_cast<uint32_t>(row);
    const uint32_t b = divP.div(n);
    const uint32_t r = n - b * static_cast<uint32_t>(P);
    const uint32_t c = divT1.div(r);
    const uint32_t t = r - c * static_cast<uint32_t>(T1);
    return t < static_cast<uint32_t>(T) && c >= static_cast<uint32_t>(npad);
  }
  // (b, t, f) of a valid row
  __host__ __device__ void coords(int64_t row, int32_t& b, int32_t& t, int32_t& f) const {
    const uint32_t n = static_cast<uint32_t>(row);
    const uint32_t bb = divP.div(n);
    const uint32_t r = n - bb * static_cast<uint32_t>(P);
    const uint32_t c = divT1.div(r);
    b = static_cast<int32_t>(bb);
    t = static_cast<int32_t>(r - c * static_cast<uint32_t>(T1));
    f = static_cast<int32_t>(c) - npad;
  }
  __host__ __device__ int64_t row_of(int32_t b, int32_t t, int32_t f) const {
    return static_cast<int64_t>(b) * P + static_cast<int64_t>(f + npad) * T1 + t;
  }
};

inline PlaneGeom make_geom(int B, int T, int F, int npad) {
  PlaneGeom g{};
  g.B = B;
  g.T = T;
  g.F = F;
  g.npad = npad;
  g.T1 = T + 1;
  g.P = static_cast<int64_t>(F + npad) * g.T1;
  g.Npos = static_cast<int64_t>(B) * g.P + static_cast<int64_t>(npad) * g.T1;
  g.Nalloc = (g.Npos + 127) / 128 * 128;
  g.n_tiles = g.Nalloc / 128;
  if (g.Nalloc >= (1ll << 31)) throw Error(1, "slot batch too large for one plane (2^31 rows)");
  g.divP = make_fastdiv(static_cast<uint32_t>(g.P));
  g.divT1 = make_fastdiv(static_cast<uint32_t>(g.T1));
  return g;
}

#define CNRX_CUDA(call)                                                                                    \
  do {                                                                                                     \
    cudaError_t e_ = (call);                                                                               \
    if (e_ != cudaSuccess)                                                                                 \
      throw ::cnrx::Error(4, std::string("CUDA error in ") + #call + ": " + cudaGetErrorString(e_));       \
  } while (0)

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw Error(1, msg);
}


// Launch `kernel` with programmatic stream serialization (PDL) unless CNRX_NO_PDL is set; the kernel
// must call pdl_wait() (sm100.cuh) before reading or writing activations.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  static const bool no_pdl = std::getenv("CNRX_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CNRX_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// Raise a kernel's dynamic shared-memory limit to at least `bytes` on the CURRENT device (function
// attributes are per device: a plan on another device, or another thread, must not rely on a cache
// filled elsewhere).  Process-wide cache keyed by (device, function).
void ensure_smem_attr(const void* func, int bytes);
}  // namespace cnrx
