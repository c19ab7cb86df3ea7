// ffma2_probe.cu — fp32 CUDA-core throughput on a B200: scalar FFMA vs packed FFMA2 / FMUL2, and the
// bit-exact conv inner step (separately rounded product then sum) as scalar FMUL+FADD vs packed
// FMUL2 + FFMA2(m, 1, acc).  16 independent accumulator chains per thread (acc += acc * w), 8 warps x 4 CTAs per SM.
// Build: nvcc -std=c++17 -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a ffma2_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t f2u(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 u2f(uint64_t a) { return *reinterpret_cast<float2*>(&a); }

template <int MODE>
__global__ void __launch_bounds__(256) probe(float* out, int iters, float one_, float xv) {
  float2 acc[8];
  float a1[16];
  for (int i = 0; i < 8; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int i = 0; i < 16; ++i) a1[i] = threadIdx.x * 1e-3f + i;
  const float2 one = make_float2(one_, one_);
  const float2 w = make_float2(xv * 0.999f, xv * 1.001f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // scalar FFMA: 16 MACs
        a1[2 * i] = fmaf(a1[2 * i], w.x, a1[2 * i]);
        a1[2 * i + 1] = fmaf(a1[2 * i + 1], w.y, a1[2 * i + 1]);
      } else if (MODE == 1) {  // FFMA2: 16 MACs
        uint64_t r;
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(acc[i])), "l"(f2u(w)), "l"(f2u(acc[i])));
        acc[i] = u2f(r);
      } else if (MODE == 2) {  // scalar FMUL + FADD: 16 separately rounded MACs
        a1[2 * i] = __fadd_rn(a1[2 * i], __fmul_rn(a1[2 * i], w.x));
        a1[2 * i + 1] = __fadd_rn(a1[2 * i + 1], __fmul_rn(a1[2 * i + 1], w.y));
      } else {  // FMUL2 + FFMA2(m, one, acc): 16 separately rounded MACs
        uint64_t m, r;
        asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(f2u(acc[i])), "l"(f2u(w)));
        asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(m), "l"(f2u(one)), "l"(f2u(acc[i])));
        acc[i] = u2f(r);
      }
    }
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
  for (int i = 0; i < 16; ++i) s += a1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const char* names[4] = {"FFMA (fused)", "FFMA2 (fused)", "FMUL+FADD (bit-exact)", "FMUL2+FFMA2(1) (bit-exact)"};
  const int iters = 20000;
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      const dim3 grid(148 * 4);
      if (mode == 0) probe<0><<<grid, 256>>>(out, iters, 1.f, 1e-6f);
      if (mode == 1) probe<1><<<grid, 256>>>(out, iters, 1.f, 1e-6f);
      if (mode == 2) probe<2><<<grid, 256>>>(out, iters, 1.f, 1e-6f);
      if (mode == 3) probe<3><<<grid, 256>>>(out, iters, 1.f, 1e-6f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double macs = 148.0 * 4 * 256 * iters * 16.0;
      if (rep == 1)
        printf("%-28s %.3f ms  %.2f T MAC/s  (%.1f MAC/clk/SM at the %d MHz max clock)\n", names[mode], ms,
               macs / ms * 1e-9, macs / (ms * 1e-3) / 148.0 / (clk_khz * 1e3), clk_khz / 1000);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
