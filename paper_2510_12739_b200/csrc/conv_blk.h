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

// The CoNet interaction + LLR head folded into the last residual blocks' conv2 epilogues (fused_head on
// the fused-block program): the last blocks of the subnetworks run as one launch per subnetwork, in fold
// order.  Launch k >= 1 reads the fold so far -- the 16-bit output plane of subnetwork 0 (k = 1, its
// step-0 BN / ReLU applied on load) or the fp32 partial-fold plane of launch k - 1 -- and combines it with
// its own output exactly as head.cu's fold does (fp32, the 16-bit-rounded subnetwork output):
//   acc = prev (op) y; [acc = fma(acc, s, t)]; [relu]
// Mid launches (EPI 1) store acc as an fp32 partial; the last (EPI 2) runs the 1x1 head on it (fp32, the
// summation order of head.cu's CUDA-core GEMV) and writes the LLRs.  The fold runs on three extra warps
// that consume the conv2 tile the epilogue warps staged, so those keep their plain per-tile work.
// network.hpp:534-559.
struct BlkFold {
  CUtensorMap opnd_map;      // (k = 1) subnetwork 0's 16-bit output plane, 63-row boxes (128B swizzle)
  const float* opnd_part;    // (k >= 2) fp32 partial-fold buffer of launch k - 1 (conv_blk64_part_bytes)
  float* pout_part;          // (EPI 1) this launch's fp32 partial-fold buffer
  const float* s_prev;       // (16-bit operand) fold step 0's BN scale / shift, nullable
  const float* t_prev;
  const float* s;            // this step's BN, nullable
  const float* t;
  const float* head_w;       // (EPI 2) [64][nb] fp32, reference 1x1 layout
  const float* head_b;       // [nb]
  float* llr;                // [B,T,F,nb]
  int32_t relu_prev, op, relu, opnd_f32, nb;
  int32_t dbg;               // experiments (CNRX_FOLD_DEBUG): bit 0 no operand loads, 1 no head, 2 no partial store
};

struct BlkLaunch {
  BlkGroup g[4];
  PlaneGeom geo;
  int64_t n_tiles;         // 63-row output tiles
  int32_t ngroups, win_alloc, xstages, relu_in;
  int32_t epi;             // 0: store y; 1 / 2: interaction fold (mid / last + head), ngroups == 1
  BlkFold fold;
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
// fold operand / output: `opnd` subnetwork 0's 16-bit plane (opnd_f32 = 0) or a partial-fold buffer;
// `pout` (EPI 1) a partial-fold buffer.  Partial-fold buffers are tile-major: per 63-row output tile one
// 16 KB block of fp32 [64 rows][64 channels], moved with plain bulk copies.
size_t conv_blk64_part_bytes(int64_t nalloc);
void conv_blk64_make_fold_maps(const void* opnd, bool opnd_f32, void* pout, int64_t nalloc, BlkFold* f);
// largest x-window ring depth (<= 6) that fits in shared memory, 0 if none
int conv_blk64_xstages(int win_alloc, int relu_in, int epi = 0);
size_t conv_blk64_smem_bytes(int xstages, int win_alloc, int relu_in, int epi = 0);
const char* conv_blk64_launch(const BlkLaunch& L, int num_sms, cudaStream_t stream);

}  // namespace cnrx
