// conv_blk.h — launch interface of the fused pre-activation residual block kernel (conv_blk.cu):
//   y = conv2(relu(bn2(conv1(relu?(x))))) + x      (64 channels, 3x3, the MRB block of network.hpp:451-465)
// with conv1's output kept in shared memory instead of a plane in HBM.
#pragma once
#include <cuda.h>

#include "common.h"

namespace cnrx {

struct BlkGroup {
  CUtensorMap in_map;      // x plane [Nalloc][64], 32-row boxes (conv1 window and the residual)
  CUtensorMap out_map;     // y plane, 63-row boxes (TMA store of one tile)
  const uint32_t* wimg1;   // conv_ws64_pack_weights images (BN folded) of conv1 and conv2
  const uint32_t* wimg2;
  const float* bias1;      // [64] conv1 bias with bn2 folded in (followed by ReLU)
  const float* bias2;      // [64]
  int32_t dil, halo;
};

struct BlkLaunch {
  BlkGroup g[4];
  PlaneGeom geo;
  int64_t n_tiles;         // 63-row output tiles
  int32_t ngroups, win_alloc, xstages, relu_in;
  int32_t fp16;             // planes and weights are fp16 (CNRX_FP16 plans), else bf16
  unsigned long long* trace;  // debug: per-role clock64 totals (kBlkTrace*)
};
enum : int {
  kBlkTraceProd = 0, kBlkTraceM1In, kBlkTraceM1Acc, kBlkTraceM2In, kBlkTraceM2Acc, kBlkTraceE1Full, kBlkTraceE1W,
  kBlkTraceE2Full, kBlkTraceTiles, kBlkTraceTotal, kBlkTraceRelu, kBlkTraceE1Fence, kBlkTraceN
};
// slots 12..15: CTA window (sm100.cuh trace_cta_window); 16..21: epilogue phases (TMEM drain, combine, store)
enum : int { kBlkTraceE1Drain = 16, kBlkTraceE1Comb, kBlkTraceE1Store, kBlkTraceE2Drain, kBlkTraceE2Comb,
             kBlkTraceE2Store, kBlkTraceSlots };

int64_t conv_blk64_tiles(int64_t nalloc);
int conv_blk64_win_alloc(int halo);
bool conv_blk64_supported_halo(int halo);
void conv_blk64_make_maps(const void* in, const void* out, int64_t nalloc, BlkGroup* g);
// largest x-window ring depth (<= 6) that fits in shared memory, 0 if none
int conv_blk64_xstages(int win_alloc, int relu_in);
size_t conv_blk64_smem_bytes(int xstages, int win_alloc, int relu_in);
const char* conv_blk64_launch(const BlkLaunch& L, int num_sms, cudaStream_t stream);

}  // namespace cnrx
