// conv_x3.h — launch interface of the split-precision tensor-core convolution (conv_x3.cu).
//
// CNRX_BF16X3 / CNRX_FP16X3 plans carry every activation value v as a pair of 16-bit numbers
// (hi = round16(v), lo = round16(v - hi)), stored side by side in a plane row of 2C 16-bit values:
// [hi 0..C-1 | lo 0..C-1] (the same bytes as fp32).  Weights are split the same way, and a conv is
// three tensor-core products per K-step, hi*Whi + hi*Wlo + lo*Whi, accumulated in fp32 in TMEM (the
// dropped lo*Wlo term is 2^-16 (bf16) / 2^-22 (fp16) of the product).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.h"
#include "conv_tc.h"

namespace cnrx {

constexpr int kX3MaxGroups = 4;

struct X3Group {
  CUtensorMap map[4];               // input plane: hi chunk 0 (<= 64 ch), hi chunk 1, lo chunk 0, lo chunk 1
  const uint8_t* wimg;              // per tap: [hi: chunk0 COUT rows | chunk1 COUT rows][lo: same], swizzled
  const float* bias;                // [COUT] (BN folded in)
  const __nv_bfloat16* res;         // residual split plane [Nalloc][2*COUT] or nullptr
  __nv_bfloat16* out;               // output split plane [Nalloc][2*COUT]
  __nv_bfloat16* out2;              // optional pre-activated copy relu(v*s2 + t2), split, or nullptr
  const float* s2;                  // nullable
  const float* t2;
  int32_t relu;
  int32_t dil;
  int32_t halo;                     // (T+1)*dil + 1, 0 for 1x1
  int32_t nb;                       // LLR head launches: bits per RE
  float* llr;                       // LLR head (3x3 output conv): fp32 [B,T,F,nb], valid rows only, instead of a plane
};

struct X3Launch {
  X3Group g[kX3MaxGroups];
  PlaneGeom geo;
  int32_t ngroups;
  int32_t stages;      // window pipeline depth
  int32_t win_alloc;   // rows per window stage (multiple of 32)
  int32_t nslots;      // weight-tap slots in shared memory; == taps: weights resident for the CTA's life
  int32_t fp16;        // 16-bit format: fp16 (else bf16)
  int32_t relu_in;     // the input is relu(plane): applied to each window pair in shared memory (ReLU warps)
  unsigned long long* trace;  // debug (CNRX_TRACE): per-role clock64 totals, conv_tc.h kTrace* indices
};

bool conv_x3_supported(int cin, int cout, int ks);
size_t conv_x3_wimg_bytes(int cin, int cout, int ks);
// w: fp32 [ks,ks,cin_real,cout_real] (reference layout), scaled per output channel by `scale` (nullable)
void conv_x3_pack_weights(const float* w, int ks, int cin_real, int cout_real, const float* scale, int cin, int cout,
                          bool fp16, uint8_t* img);
// Tensor maps (32-row boxes) over the hi / lo K-chunks of a split plane [nalloc][2*cin]; null plane: zeroed.
void conv_x3_make_maps(const void* plane, int64_t nalloc, int cin, CUtensorMap* maps);
// Pick the window depth and weight-slot count that fit shared memory (weights resident when they fit).
bool conv_x3_config(int cin, int cout, int ks, int win_alloc, int* stages, int* nslots);
size_t conv_x3_smem_bytes(int cin, int cout, int ks, int stages, int win_alloc, int nslots);
const char* conv_x3_launch(int cin, int cout, int ks, const X3Launch& L, int num_sms, cudaStream_t stream);

}  // namespace cnrx
