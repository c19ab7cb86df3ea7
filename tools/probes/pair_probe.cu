// pair_probe.cu — pins the cta_group::2 (CTA pair) UMMA semantics this repo relies on:
//   * a cluster of 2 CTAs; the leader (rank 0) issues tcgen05.mma.cta_group::2 with M = 256, N = 96;
//   * A rows 0..127 come from rank 0's shared memory, rows 128..255 from rank 1's (same smem offset);
//   * B (N x K, K-major) is split by N: rank 0 holds rows 0..47, rank 1 rows 48..95 (same offset);
//   * D lands in each CTA's own TMEM: rank r holds rows 128r..128r+127, all 96 columns;
//   * tcgen05.commit ... multicast::cluster arrives on the barrier at the same offset in both CTAs.
// Prints max |D - A B^T| over the full 256 x 96 result (expected 0: small integers, exact in fp32).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 -I../../paper_2510_12739_b200/csrc pair_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace cnrx;

constexpr int M = 256, N = 96, K = 16;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pair_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];  // 128 rows x 16 bf16 (32 B), no swizzle, core 8x16B
  __shared__ __align__(1024) uint8_t sB[48 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_rank();
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  // fill A rows (this CTA's 128) and B rows (this CTA's 48) in the no-swizzle K-major core-matrix layout:
  // element (row, k) at ((row/8) * (K/8) + k/8) * 128 + (row%8) * 16 + (k%8) * 2
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    const int row = i / K, k = i % K;
    const __nv_bfloat16 v = A[(rank * 128 + row) * K + k];
    *reinterpret_cast<__nv_bfloat16*>(sA + ((row / 8) * (K / 8) + k / 8) * 128 + (row % 8) * 16 + (k % 8) * 2) = v;
  }
  for (int i = tid; i < 48 * K; i += blockDim.x) {
    const int row = i / K, k = i % K;
    const __nv_bfloat16 v = B[(rank * 48 + row) * K + k];
    *reinterpret_cast<__nv_bfloat16*>(sB + ((row / 8) * (K / 8) + k / 8) * 128 + (row % 8) * 16 + (k % 8) * 2) = v;
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(128)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = slot;
  if (rank == 0 && tid == 0) {
    // no-swizzle K-major: LBO = byte distance between the two K core matrices (128), SBO = between 8-row groups (256)
    const uint64_t ad = (make_sdesc(smem_u32(sA), 256, kSwizzleNone, 0) & ~(0x3FFFull << 16)) | (static_cast<uint64_t>(128 >> 4) << 16);
    const uint64_t bd = (make_sdesc(smem_u32(sB), 256, kSwizzleNone, 0) & ~(0x3FFFull << 16)) | (static_cast<uint64_t>(128 >> 4) << 16);
    const uint32_t idesc = idesc_bf16_f32(M, N);
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tbase),
        "l"(ad), "l"(bd), "r"(idesc), "r"(0)
        : "memory");
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     smem_u32(&bar)),
                 "h"(static_cast<uint16_t>(3))
                 : "memory");
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // each CTA: 128 lanes x 96 columns of its own TMEM
  for (int c = 0; c < N; c += 32) {
    uint32_t r[32];
    tmem_ld32(tbase + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) D[(rank * 128 + warp * 32 + lane) * N + c + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(128) : "memory");
}

int main() {
  std::vector<__nv_bfloat16> hA(M * K), hB(N * K);
  std::vector<float> fA(M * K), fB(N * K);
  for (int i = 0; i < M * K; ++i) {
    fA[i] = static_cast<float>((i * 7 % 11) - 5);
    hA[i] = __float2bfloat16(fA[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    fB[i] = static_cast<float>((i * 5 % 9) - 4);
    hB[i] = __float2bfloat16(fB[i]);
  }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, N * K * 2);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, M * N * 4);
  pair_kernel<<<2, 128>>>(dA, dB, dD);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> hD(M * N);
  cudaMemcpy(hD.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += fA[m * K + k] * fB[n * K + k];
      const double err = std::fabs(ref - hD[m * N + n]);
      if (err > maxerr) maxerr = err;
      if (err > 0 && bad < 5) {
        printf("mismatch m=%d n=%d got %f want %f\n", m, n, hD[m * N + n], ref);
        ++bad;
      }
    }
  printf("cta_group::2 M=256 N=96: max |D - A B^T| = %g\n", maxerr);
  return maxerr == 0 ? 0 : 2;
}
