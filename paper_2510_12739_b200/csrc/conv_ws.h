// conv_ws.h — launch interface of the weights-stationary (A in TMEM) 3x3 64->64 conv (conv_ws.cu).
#pragma once
#include <cuda.h>

#include "common.h"

namespace cnrx {

struct WsGroup {
  CUtensorMap in_map;    // input plane [Nalloc][64], 32-row boxes (activation window, B operand)
  CUtensorMap res_map;   // residual plane, 32-row boxes
  CUtensorMap out_map;   // output plane, 127-row boxes (TMA store of one tile)
  CUtensorMap out2_map;  // pre-activated copy, 127-row boxes
  const uint32_t* wimg;  // conv_ws64_pack_weights image: [24 blocks][128 lanes][8 x u32]
  const float* bias;     // [64] (BN folded in)
  const float* s2;       // out2 = relu(v*s2 + t2) (null: relu(v))
  const float* t2;
  int32_t relu, dil, halo, res_map_valid, out2_map_valid;
  int32_t relu_in;       // apply ReLU to the input window in shared memory (consumer-side pre-activation)
};

// Fused CoNet interaction + LLR head (kWsHead launches: the last conv of every subnetwork in one
// launch, clusters of ngroups CTAs, CTA rank r computing fold operand r of the same tile).  Ranks >= 1
// copy their output tile into rank 0's shared memory (distributed shared memory); rank 0 folds
//   z = [aff_0][relu_0](y_0) (op_1) y_1 [aff_1][relu_1] ...
// (head.cu's fold, fp32), rounds z to bf16 and runs the 1x1 head on the tensor core.
struct WsHead {
  const float* aff_s[3];  // per fold step: eval BN scale / shift, or null
  const float* aff_t[3];
  int32_t op[3];          // PW_MUL / PW_ADD for steps >= 1
  int32_t relu[3];
  const float* w;         // [64][nb] head weights (reference 1x1 layout)
  const float* b;         // [nb]
  float* llr;             // [B,T,F,nb], set per call
  int32_t ns, nb;
};

struct WsLaunch {
  WsGroup g[4];
  WsHead head;
  int32_t head_on;
  PlaneGeom geo;
  int64_t n_tiles;   // 127-row output tiles
  int32_t ngroups, stages, win_alloc;
  int32_t fp16;      // planes and weights are fp16 (CNRX_FP16 plans), else bf16
  int32_t debug;     // experiments only (CNRX_WS_DEBUG): bit 0 skip staging writes + stores, bit 1 skip input ReLU pass;
                     // fused head: bit 4 trace rank 1 instead of rank 0, bit 5 skip the head UMMAs, bit 6 skip
                     // the fold pass, bit 7 skip the DSMEM exchange (results invalid with bits 5-7)
  unsigned long long* trace;  // debug: per-role clock64 totals (kTrace* in conv_tc.h + kWsTrace*)
};
enum : int { kWsTraceCombine = 8, kWsTraceStageWait, kWsTraceWrite, kWsTraceN };
// slots 12..15 hold the CTA window (sm100.cuh trace_cta_window); 16, 17: MMA loop-back and commit cycles
enum : int { kWsTraceLoop = 16, kWsTraceCommit = 17, kWsTraceSlots = 18 };

size_t conv_ws64_wimg_bytes();
// w: fp32 [3,3,64,64] reference layout, scale: per-output-channel BN fold (nullable)
void conv_ws64_pack_weights(const float* w, const float* scale, bool fp16, uint32_t* img);
void conv_ws64_make_maps(const void* in, const void* res, const void* out, const void* out2, int64_t nalloc,
                         WsGroup* g);
size_t conv_ws64_smem_bytes(int stages, int win_alloc);
size_t conv_ws64_head_smem_bytes(int stages, int win_alloc);
int conv_ws64_win_alloc(int halo);
int64_t conv_ws64_tiles(int64_t nalloc);
const char* conv_ws64_launch(const WsLaunch& L, int num_sms, cudaStream_t stream);

}  // namespace cnrx
