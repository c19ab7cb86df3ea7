// umma_probe.cu — pins the hardware facts the CoNet-Rx conv kernels rely on (run on a B200):
//  1. UMMA K-major SW128 A operand addressed at an arbitrary ROW offset inside a TMA-loaded window:
//     which descriptor base_offset value makes it read the right rows (0 or row&7)?
//  2. TMA zero fill for negative / past-the-end row coordinates.
//  3. tcgen05.mma (SS, M=128, K=16) throughput for N = 64 / 96 / 128 / 256, aligned vs. shifted A.
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I../../paper_2510_12739_b200/csrc
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace cnrx;

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                              \
    }                                                                                       \
  } while (0)

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static CUtensorMap make_map(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, uint32_t box_cols,
                            CUtensorMapSwizzle sw) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "tensor map encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

// ------------------------------------------------------------------------------------------
// 1+2: shift semantics. A window of 192 rows loaded from row coordinate `row0` (may be negative).
// For each case c: shift s = c % 32, base-offset variant v = c / 32 (0: zero, 1: s&7).
// out[c][128][64] = A_window[s : s+128] * B^T.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 1)
    shift_probe(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int row0,
                float* out, int ncases, __nv_bfloat16* win_dump) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                  // 192 rows x 128 B = 24 KB
  uint8_t* sB = smem + 192 * 128;      // 64 rows x 128 B = 8 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar_load, 192 * 128 + 64 * 128);
    tma_load_2d(sA, &mapA, &bar_load, 0, row0);  // box is 192 rows? no: two loads of 96 rows
    tma_load_2d(sA + 96 * 128, &mapA, &bar_load, 0, row0 + 96);
    tma_load_2d(sB, &mapB, &bar_load, 0, 0);
  }
  mbar_wait(&bar_load, 0);
  // dump the (de-swizzled) window so the host can check zero fill
  for (int r = threadIdx.x; r < 192; r += blockDim.x)
    for (int ch = 0; ch < 8; ++ch) {
      const uint4 v = *reinterpret_cast<const uint4*>(sA + sw128_offset(r, ch));
      *reinterpret_cast<uint4*>(win_dump + r * 64 + ch * 8) = v;
    }
  const uint32_t idesc = idesc_bf16_f32(128, 64);
  uint32_t phase = 0;
  for (int c = 0; c < ncases; ++c) {
    const int s = c % 32, v = c / 32;
    if (threadIdx.x == 0) {
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t a_start = smem_u32(sA) + s * 128 + kk * 32;
        const uint32_t b_start = smem_u32(sB) + kk * 32;
        const uint64_t ad = make_sdesc(a_start, 1024, kSwizzle128, v ? (s & 7) : 0);
        const uint64_t bd = make_sdesc(b_start, 1024, kSwizzle128, 0);
        umma_bf16(tbase, ad, bd, idesc, kk > 0);
      }
      umma_commit(&bar_mma);
    }
    __syncwarp();
    mbar_wait(&bar_mma, phase);
    phase ^= 1;
    tc_fence_after();
    uint32_t r[32];
    const int row = warp * 32 + lane_id();
    for (int half = 0; half < 2; ++half) {
      tmem_ld32(tbase + ((warp * 32) << 16) + half * 32, r);
      tmem_ld_wait();
      for (int j = 0; j < 32; ++j) out[(size_t(c) * 128 + row) * 64 + half * 32 + j] = __uint_as_float(r[j]);
    }
    tc_fence_before();
    __syncthreads();
  }
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 64);
}

// ------------------------------------------------------------------------------------------
// 3: MMA throughput. Every CTA issues `iters` x 4 k-steps of M=128 x N x 16 from one thread.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 1) mma_rate(int N, int iters, int shift, long long* cycles, int nacc = 2,
                                                  int per_acc = 4) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 160 rows x 128 B
  uint8_t* sB = smem + 160 * 128;   // 256 rows x 128 B
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (160 + 256) * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N);
    const long long t0 = clock64();
    // nacc accumulators (columns N apart), per_acc consecutive MMAs into one before moving on
    int cnt = 0;
    for (int it = 0; it < iters; ++it) {
      const int sh = shift ? (it % 33) : 0;
      for (int kk = 0; kk < 4; ++kk, ++cnt) {
        const uint64_t ad = make_sdesc(smem_u32(sA) + sh * 128 + kk * 32, 1024, kSwizzle128, 0);
        const uint64_t bd = make_sdesc(smem_u32(sB) + kk * 32, 1024, kSwizzle128, 0);
        const int acc = (cnt / per_acc) % nacc;
        umma_bf16(tbase + acc * N, ad, bd, idesc, 1);
      }
    }
    umma_commit(&bar_mma);
    mbar_wait(&bar_mma, 0);
    const long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

static float bf16_to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

// ------------------------------------------------------------------------------------------
// 4: MMA throughput under concurrent LSU shared-memory traffic: warp 0 issues MMAs (M=128, N, K=16,
// SS) while warps 1..nw stream 16-byte LDS+STS over a separate 32 KB buffer.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) mma_contention(int N, int iters, int lsu_warps, long long* cycles,
                                                         unsigned long long* lsu_bytes) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;               // 160 rows x 128 B
  uint8_t* sB = smem + 160 * 128;   // 256 rows x 128 B
  uint8_t* sX = smem + (160 + 256) * 128;  // 32 KB scratch for LSU traffic
  __shared__ uint64_t bar_mma;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (160 + 256) * 128 / 16 + 2048; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp == 0) {
    if (lane_id() == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, N);
      uint64_t ad[4], bd[4];
      for (int kk = 0; kk < 4; ++kk) {
        ad[kk] = make_sdesc(smem_u32(sA) + 3 * 128 + kk * 32, 1024, kSwizzle128, 0);
        bd[kk] = make_sdesc(smem_u32(sB) + kk * 32, 1024, kSwizzle128, 0);
      }
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16(tbase + (it & 1) * 256, ad[kk], bd[kk], idesc, 1);
      }
      umma_commit(&bar_mma);
      mbar_wait(&bar_mma, 0);
      cycles[blockIdx.x] = clock64() - t0;
      done = 1;
    }
  } else if (warp <= lsu_warps) {
    // fixed work: 4096 x (LDS.128 + STS.128) per lane, timed per warp
    uint4* x = reinterpret_cast<uint4*>(sX);
    const int i = (warp - 1) * 32 + lane_id();
    const long long t0 = clock64();
    uint32_t acc = 0;
#pragma unroll 1
    for (int r = 0; r < 4096; r += 8) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = x[(i + (r + u) * 224) & 2047];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u].x += acc;
        x[(i + (r + u) * 224 + 64) & 2047] = v[u];
        acc += v[u].y;
      }
    }
    const long long t1 = clock64();
    if (lane_id() == 0) atomicAdd(lsu_bytes, static_cast<unsigned long long>(t1 - t0));
    if (acc == 0xdeadbeef) x[0].x = acc;
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------------------------------
// 5: A-from-TMEM MMA throughput (M=128, N, K=16) with optional concurrent traffic from warps 1..7:
// mode 0 none, 1 LDG.128 streaming, 2 STG.128 streaming, 3 LDS+STS, 4 TMA 2D loads (32 x 128 B boxes)
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) mma_ts_rate(int N, int iters, int mode, long long* cycles,
                                                      unsigned long long* side_bytes, const uint4* gsrc, uint4* gdst,
                                                      const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem;                      // 256 rows x 128 B = 32 KB
  uint8_t* sX = smem + 256 * 128;          // 32 KB scratch
  __shared__ uint64_t bar_mma, bar_tma;
  __shared__ uint32_t tmem_base;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar_mma, 1);
    mbar_init(&bar_tma, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp >= 4) {  // fill A region (columns 0..63) with bf16 ones: lanes of this warp's quadrant
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = 0x3f803f80u;
    for (int c = 0; c < 64; c += 8) tmem_st8(tbase + ((32 * (warp & 3)) << 16) + c, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (lane_id() == 0) {
      const uint32_t idesc = idesc_bf16_f32(128, N);
      uint64_t bd[4];
      for (int kk = 0; kk < 4; ++kk) bd[kk] = make_sdesc(smem_u32(sB) + 3 * 128 + kk * 32, 1024, kSwizzle128, 0);
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_bf16_ts(tbase + 256 + (it & 1) * (N > 128 ? 0 : 128), tbase + kk * 8, bd[kk], idesc, 1);
      }
      umma_commit(&bar_mma);
      mbar_wait(&bar_mma, 0);
      cycles[blockIdx.x] = clock64() - t0;
      done = 1;
    }
  } else {
    unsigned long long bytes = 0;
    const int tid = threadIdx.x - 32;  // 0..223
    if (mode == 1) {
      uint32_t acc = 0;
      const uint4* src = gsrc + (size_t)blockIdx.x * 65536;
      int i = tid;
      while (!done) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + ((i + u * 224) & 65535)));
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x;
        i += 8 * 224;
        bytes += 8 * 16;
      }
      if (acc == 0xdeadbeef) gdst[0].x = acc;
    } else if (mode == 2) {
      uint4* dst = gdst + (size_t)blockIdx.x * 65536;
      int i = tid;
      while (!done) {
#pragma unroll
        for (int u = 0; u < 8; ++u) dst[(i + u * 224) & 65535] = make_uint4(i, u, 0, 0);
        i += 8 * 224;
        bytes += 8 * 16;
      }
    } else if (mode == 3) {
      uint4* x = reinterpret_cast<uint4*>(sX);
      int i = tid;
      uint32_t acc = 0;
      while (!done) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = x[(i + u * 224) & 2047];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u].x += acc;
          x[(i + u * 224 + 64) & 2047] = v[u];
          acc += v[u].y;
        }
        i += 8 * 224;
        bytes += 8 * 32;
      }
    } else if (mode == 4 && tid == 0) {
      uint32_t ph = 0;
      int r = blockIdx.x * 64;
      while (!done) {
        mbar_arrive_expect_tx(&bar_tma, 8 * 32 * 128);
        for (int u = 0; u < 8; ++u) tma_load_2d(sX + u * 4096, &tmap, &bar_tma, 0, (r + u * 32) & 32767);
        mbar_wait(&bar_tma, ph);
        ph ^= 1;
        r += 256;
        bytes += 8 * 32 * 128;
      }
    }
    atomicAdd(side_bytes, bytes);
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s sm_%d%d SMs=%d\n", prop.name, prop.major, prop.minor, prop.multiProcessorCount);

  // ---- shift semantics ----
  const int ROWS = 512;
  std::vector<__nv_bfloat16> hA(ROWS * 64), hB(64 * 64);
  for (int r = 0; r < ROWS; ++r)
    for (int k = 0; k < 64; ++k) hA[r * 64 + k] = __float2bfloat16(float(((r * 7 + k * 3) % 9) - 4));
  for (int n = 0; n < 64; ++n)
    for (int k = 0; k < 64; ++k) hB[n * 64 + k] = __float2bfloat16(float(((n * 5 + k * 11) % 7) - 3));
  __nv_bfloat16 *dA, *dB, *dWin;
  float* dOut;
  const int ncases = 64;
  CK(cudaMalloc(&dA, hA.size() * 2));
  CK(cudaMalloc(&dB, hB.size() * 2));
  CK(cudaMalloc(&dOut, size_t(ncases) * 128 * 64 * 4));
  CK(cudaMalloc(&dWin, 192 * 64 * 2));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  CUtensorMap mA = make_map(dA, ROWS, 64, 96, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  CUtensorMap mB = make_map(dB, 64, 64, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  CK(cudaFuncSetAttribute(shift_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  int fails = 0;
  for (int row0 : {40, -5, ROWS - 150}) {
    shift_probe<<<1, 128, 64 * 1024>>>(mA, mB, row0, dOut, ncases, dWin);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> out(size_t(ncases) * 128 * 64);
    std::vector<__nv_bfloat16> win(192 * 64);
    CK(cudaMemcpy(out.data(), dOut, out.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(win.data(), dWin, win.size() * 2, cudaMemcpyDeviceToHost));
    auto arow = [&](int wr, int k) -> float {  // expected window content
      int gr = row0 + wr;
      if (gr < 0 || gr >= ROWS) return 0.f;
      return bf16_to_f(hA[gr * 64 + k]);
    };
    int win_bad = 0;
    for (int r = 0; r < 192; ++r)
      for (int k = 0; k < 64; ++k)
        if (bf16_to_f(win[r * 64 + k]) != arow(r, k)) ++win_bad;
    printf("row0=%d: window mismatches (TMA load/zero-fill) = %d\n", row0, win_bad);
    fails += win_bad != 0;
    for (int v = 0; v < 2; ++v) {
      int ok_shifts = 0, first_bad = -1;
      for (int s = 0; s < 32; ++s) {
        const int c = v * 32 + s;
        int bad = 0;
        for (int m = 0; m < 128 && !bad; ++m)
          for (int n = 0; n < 64; ++n) {
            float ref = 0.f;
            for (int k = 0; k < 64; ++k) ref += arow(s + m, k) * bf16_to_f(hB[n * 64 + k]);
            if (out[(size_t(c) * 128 + m) * 64 + n] != ref) {
              bad = 1;
              break;
            }
          }
        if (!bad) ++ok_shifts;
        else if (first_bad < 0) first_bad = s;
      }
      printf("  base_offset=%s : %d/32 shifts exact (first bad shift %d)\n", v ? "row&7" : "0", ok_shifts,
             first_bad);
    }
  }

  // ---- throughput ----
  long long* dCyc;
  const int nblk = prop.multiProcessorCount;
  CK(cudaMalloc(&dCyc, nblk * sizeof(long long)));
  CK(cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct Cfg { int N, shift, nacc, per; };
  for (Cfg c : {Cfg{64, 0, 1, 1}, Cfg{64, 0, 2, 1}, Cfg{64, 0, 4, 1}, Cfg{64, 0, 2, 4}, Cfg{64, 0, 2, 36},
                Cfg{64, 1, 1, 1}, Cfg{64, 1, 4, 1}, Cfg{128, 0, 1, 1}, Cfg{128, 0, 2, 1}, Cfg{96, 0, 1, 1},
                Cfg{96, 0, 4, 1}, Cfg{256, 0, 1, 1}, Cfg{32, 0, 1, 1}, Cfg{32, 0, 4, 1}}) {
      const int N = c.N, shift = c.shift;
      const int iters = 20000;
      mma_rate<<<nblk, 128, 60 * 1024>>>(N, 100, shift, dCyc, c.nacc, c.per);  // warm-up
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      mma_rate<<<nblk, 128, 60 * 1024>>>(N, iters, shift, dCyc, c.nacc, c.per);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      std::vector<long long> cyc(nblk);
      CK(cudaMemcpy(cyc.data(), dCyc, nblk * 8, cudaMemcpyDeviceToHost));
      double mean_cyc = 0;
      for (auto c : cyc) mean_cyc += c;
      mean_cyc /= nblk;
      const double flop = 2.0 * 128 * N * 16 * 4.0 * iters * nblk;
      printf("MMA M=128 N=%3d K=16 shiftedA=%d nacc=%d per_acc=%2d: %.1f cyc/MMA/SM, %.1f TFLOP/s (event %.3f ms)\n",
             N, shift, c.nacc, c.per, mean_cyc / (iters * 4.0), flop / (ms * 1e-3) / 1e12, ms);
    }
  {
    unsigned long long* dB;
    CK(cudaMalloc(&dB, 8));
    CK(cudaFuncSetAttribute(mma_contention, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
    for (int N : {64, 256})
      for (int lw : {0, 1, 2, 4, 7}) for (int iters : {0, 20000}) {
        if (iters == 0 && N == 256) continue;
        CK(cudaMemset(dB, 0, 8));
        mma_contention<<<nblk, 256, 100 * 1024>>>(N, iters, lw, dCyc, dB);
        CK(cudaDeviceSynchronize());
        std::vector<long long> cyc(nblk);
        CK(cudaMemcpy(cyc.data(), dCyc, nblk * 8, cudaMemcpyDeviceToHost));
        unsigned long long hb = 0;
        CK(cudaMemcpy(&hb, dB, 8, cudaMemcpyDeviceToHost));
        double mc = 0;
        for (auto c : cyc) mc += c;
        mc /= nblk;
        const double lsu_cyc = lw ? double(hb) / nblk / lw : 0;  // avg cycles per LSU warp
        const double lsu_bw = lw ? (4096.0 * 32 * 32 * lw) / lsu_cyc : 0;  // bytes (LDS+STS) per cycle per SM
        printf("contention N=%3d iters=%d lsu_warps=%d: %.1f cyc/MMA (MMA span %.0f cyc), LSU warp span %.0f cyc, "
               "LSU smem %.1f B/cyc/SM while running\n", N, iters, lw, iters ? mc / (iters * 4.0) : 0.0, mc, lsu_cyc,
               lsu_bw);
      }
  }
  {
    unsigned long long* dB;
    CK(cudaMalloc(&dB, 8));
    uint4 *gs, *gd;
    CK(cudaMalloc(&gs, size_t(nblk) * 65536 * 16));
    CK(cudaMalloc(&gd, size_t(nblk) * 65536 * 16));
    CK(cudaMemset(gs, 0, size_t(nblk) * 65536 * 16));
    CUtensorMap tm = make_map(gs, 32768, 64, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B);
    CK(cudaFuncSetAttribute(mma_ts_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
    const char* names[5] = {"none", "LDG.128 nc", "STG.128", "LDS+STS", "TMA 2D load"};
    for (int N : {32, 64, 96, 128, 256})
      for (int mode = 0; mode < (N < 128 ? 1 : 5); ++mode) {
        const int iters = 20000;
        CK(cudaMemset(dB, 0, 8));
        mma_ts_rate<<<nblk, 256, 80 * 1024>>>(N, iters, mode, dCyc, dB, gs, gd, tm);
        CK(cudaDeviceSynchronize());
        std::vector<long long> cyc(nblk);
        CK(cudaMemcpy(cyc.data(), dCyc, nblk * 8, cudaMemcpyDeviceToHost));
        unsigned long long hb = 0;
        CK(cudaMemcpy(&hb, dB, 8, cudaMemcpyDeviceToHost));
        double mc = 0;
        for (auto c : cyc) mc += c;
        mc /= nblk;
        printf("A-in-TMEM N=%3d side=%-12s: %.1f cyc/MMA, side traffic %.1f B/cyc/SM\n", N, names[mode],
               mc / (iters * 4.0), double(hb) / nblk / mc);
      }
  }
  printf("probe fails=%d\n", fails);
  return fails ? 2 : 0;
}
