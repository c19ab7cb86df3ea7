// m64_probe.cu — tcgen05.mma kind::f16 with A in TMEM (the weights-stationary conv form) at M = 64 vs
// M = 128, cta_group::1 (run on a B200):
//   1. issue rate: cycles per UMMA for (M, N) in {128, 64} x {64, 128};
//   2. lane mapping: which TMEM lanes an M = 64 UMMA reads A rows from and writes D rows to.
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I../../paper_2510_12739_b200/csrc m64_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "elem16.cuh"
#include "sm100.cuh"

using namespace cnrx;

#define CK(x)                                                                                 \
  do {                                                                                        \
    cudaError_t e = (x);                                                                      \
    if (e != cudaSuccess) {                                                                   \
      fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                                \
    }                                                                                         \
  } while (0)

// idesc: D f32, A/B bf16, K-major, N, M
__host__ __device__ constexpr uint32_t idesc_mn(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// rate: one thread issues `iters` x 4 UMMAs (K = 64) of shape M x N, A from TMEM columns 0..31, B from smem
// lane map (iters == 0): A lane l holds the value l + 1 (bf16, exact for l < 255) in every K column, B rows are all
// ones, one UMMA of M = 64, N = 8 into D columns 256..263; every thread of the 4 warps reads its lane's D
// column 256: D = 16 * (A lane feeding that row + 1) for K = 16, or 0 where no row lands.
__global__ void __launch_bounds__(128, 1) probe(int M, int N, int iters, long long* cycles, float* lanemap) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // B: 256 rows x 128 B of bf16 ones (K-major, SW128 is irrelevant for constant data)
  for (int i = threadIdx.x; i < 256 * 128 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  {  // A (TMEM columns 0..31, K = 64 bf16): lane value = lane index
    const uint32_t l = static_cast<uint32_t>(32 * warp + lane);
    const uint32_t v = pack2<false>(static_cast<float>(l + 1), static_cast<float>(l + 1));
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = v;
    for (int c = 0; c < 32; c += 8) tmem_st8(tbase + (static_cast<uint32_t>(32 * warp) << 16) + c, r);
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int c = 256; c < 512; c += 8) tmem_st8(tbase + (static_cast<uint32_t>(32 * warp) << 16) + c, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {
    const uint64_t bd = make_sdesc(smem_u32(smem), 1024, kSwizzle128, 0);
    if (iters == 0) {
      umma_f16_ts(tbase + 256, tbase, bd, idesc_mn(M, 8), 0);
      umma_commit(&bar);
      mbar_wait(&bar, 0);
    } else {
      const uint32_t idesc = idesc_mn(M, N);
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_f16_ts(tbase + 256 + (it & 1) * 128, tbase + kk * 8, bd + static_cast<uint64_t>(kk * 2), idesc, 1);
      }
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      cycles[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (iters == 0) {
    uint32_t r[8];
    tmem_ld8(tbase + (static_cast<uint32_t>(32 * warp) << 16) + 256, r);
    tmem_ld_wait();
    lanemap[32 * warp + lane] = __uint_as_float(r[0]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  long long* dc;
  float* dl;
  CK(cudaMalloc(&dc, 148 * sizeof(long long)));
  CK(cudaMalloc(&dl, 128 * sizeof(float)));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
  const int shapes[6][2] = {{128, 64}, {64, 64}, {128, 128}, {64, 128}, {128, 32}, {64, 32}};
  for (auto& s : shapes) {
    const int iters = 2000;
    probe<<<148, 128, 40 * 1024>>>(s[0], s[1], iters, dc, dl);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    long long hc[148];
    CK(cudaMemcpy(hc, dc, sizeof hc, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (long long c : hc) avg += static_cast<double>(c);
    avg /= 148.0;
    printf("A-in-TMEM M=%3d N=%3d : %.1f cycles per UMMA (K=16), %.0f MAC/clk\n", s[0], s[1], avg / (4.0 * iters),
           s[0] * s[1] * 16.0 / (avg / (4.0 * iters)));
  }
  probe<<<1, 128, 40 * 1024>>>(64, 8, 0, dc, dl);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  float hl[128];
  CK(cudaMemcpy(hl, dl, sizeof hl, cudaMemcpyDeviceToHost));
  printf("M=64 lane map (TMEM lane: A lane feeding its D row = D / 16 - 1; -1 = nothing written):\n");
  for (int l = 0; l < 128; ++l) printf("%d:%g%s", l, hl[l] / 16.f - 1.f, (l % 16 == 15) ? "\n" : " ");
  return 0;
}
