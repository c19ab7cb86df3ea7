// conv_tc.h — launch interface of the tcgen05 implicit-GEMM convolution (conv_tc.cu).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.h"

namespace cnrx {

constexpr int kTcMaxGroups = 4;
// batches up to this many slots run fused residual blocks (conv_blk.cu) when the plan has them (CNRX_BLK=0/1 forces)
constexpr int kBlkAutoMaxBatch = 1 << 30;  // every batch: measured faster sustained at B = 256 (less HBM traffic -> higher power-capped clock)

// One convolution of a grouped launch (e.g. the same layer of the three CoNet subnetworks).
struct TcGroup {
  CUtensorMap map[2];               // input plane, K-chunk 0 (<=64 ch) and chunk 1 (remaining ch)
  CUtensorMap res_map;              // staged epilogue (COUT <= 64): residual plane, 32-row boxes
  CUtensorMap out_map;              // staged epilogue: primary output plane, 32-row boxes
  CUtensorMap out2_map;             // staged epilogue: pre-activated copy
  // conv_pair.cu staged epilogue (96-ch planes as 64 + 32 channel chunks, 128-row boxes): residual
  // loads and output / pre-activated-copy stores by TMA
  CUtensorMap pres[2], pout[2], pout2[2];
  const uint8_t* wimg;              // weights, pre-swizzled smem image: [tap][chunk][COUT rows]
  const float* bias;                // [COUT] (BN folded in)
  const __nv_bfloat16* res;         // residual plane [Nalloc][COUT] or nullptr
  __nv_bfloat16* out;               // primary output plane [Nalloc][COUT]
  __nv_bfloat16* out2;              // optional pre-activated copy for the next conv, or nullptr
  const float* s2;                  // out2 = relu(v*s2 + t2) (nullptr: relu(v))
  const float* t2;
  int32_t relu;                     // relu on the primary output (after bias / residual)
  int32_t dil;                      // dilation along F
  int32_t halo;                     // window halo rows = (T+1)*dil + 1 (0 for 1x1)
  int32_t nb;                       // LLR head launches: bits per RE
  float* llr;                       // LLR head (3x3 output conv): fp32 [B,T,F,nb], valid rows only, instead of a plane
};

struct TcLaunch {
  TcGroup g[kTcMaxGroups];
  PlaneGeom geo;
  int32_t ngroups;
  int32_t stages;                   // window pipeline depth
  int32_t win_alloc;                // rows allocated per window stage (max over groups, 8-aligned)
  int32_t flags;                    // bit 0: a group has a residual, bit 1: a group writes out2
  int32_t fp16;                     // planes and weights are fp16 (CNRX_FP16 plans), else bf16
  // debug: when non-null each CTA adds per-role clock64 totals (see kTrace* indices)
  unsigned long long* trace;
};
enum : int { kTraceProdWaitEmpty = 0, kTraceMmaWaitFull, kTraceMmaWaitTmem, kTraceMmaIssue, kTraceEpiWaitFull,
             kTraceEpiWork, kTraceTiles, kTraceTotal, kTraceN };

// Shared memory the kernel needs for (cin, cout, ks) with `stages` window stages of `win_alloc` rows.
size_t conv_tc_smem_bytes(int cin, int cout, int ks, int stages, int win_alloc, int flags);
bool conv_tc_supported(int cin, int cout, int ks);
// Enqueue one grouped launch; grid = min(#SMs, ngroups * tiles).  Returns the kernel name.
const char* conv_tc_launch(int cin, int cout, int ks, const TcLaunch& L, int num_sms, cudaStream_t stream);

// Host helpers to build the operand layouts the kernel expects.
// Byte size of the weight image for (cin, cout, ks).
size_t conv_tc_wimg_bytes(int cin, int cout, int ks);
// w: fp32 [ks,ks,cin_real,cout_real] (reference layout, kernels.hpp:32), scaled per output channel
// by `scale` (nullable, folded BN); written as bf16 (fp16 if `fp16`) into `img` (host buffer of
// conv_tc_wimg_bytes).
void conv_tc_pack_weights(const float* w, int ks, int cin_real, int cout_real, const float* scale, int cin,
                          int cout, bool fp16, uint8_t* img);
// Tensor maps for the K-chunks (<= 64 + rest channels) of a plane [nalloc][cin] bf16, boxes of
// `box_rows` rows; a null plane yields zeroed maps.
void conv_tc_make_maps(const void* plane, int64_t nalloc, int cin, int box_rows, CUtensorMap* maps);
// Single-chunk (<= 64 channels) plane map with 32-row boxes for the staged epilogue (residual load,
// output stores); a null plane yields a zeroed map.
void conv_tc_make_row_map(const void* plane, int64_t nalloc, int c, CUtensorMap* map);
// True when (cin, cout) uses the staged (TMA-load residual / TMA-store outputs) epilogue.
bool conv_tc_staged(int cin, int cout);

}  // namespace cnrx
