// head.h — TMA-streamed fusion tail + LLR head (head.cu).
#pragma once
#include <cuda.h>

#include "common.h"
#include "kernels.h"

namespace cnrx {

constexpr int kHeadMaxPlanes = 4;

struct HeadLaunch {
  CUtensorMap maps[kHeadMaxPlanes];  // operand planes [Nalloc][C] bf16, 128-row boxes
  PlaneGeom geo;
  const float* aff_s[kHeadMaxPlanes];  // per fold step: eval BN scale / shift, or null
  const float* aff_t[kHeadMaxPlanes];
  int32_t op[kHeadMaxPlanes];          // PW_MUL / PW_ADD for steps >= 1
  int32_t relu[kHeadMaxPlanes];
  const float* head_w;                 // [C][nb]
  const float* head_b;                 // [nb]
  float* llr;                          // [B,T,F,nb]
  int32_t ns, nb, stages;
  int32_t fp16;                        // operand planes are fp16 (else bf16)
  int32_t tc_head;                     // C == 64: GEMV on the tensor core over bf16-rounded z
  int32_t split;                       // split planes (CNRX_*X3 plans): operand i = hi (maps[i]) + lo (lo_maps[i])
  CUtensorMap lo_maps[kHeadMaxPlanes];
  // C = 96: each tile row is two swizzled boxes, channels [0, 64) (maps / lo_maps, 128B swizzle) and
  // [64, 96) (these, 64B swizzle), so the consumers' 16-byte reads of 32 rows spread over all banks
  CUtensorMap maps_c1[kHeadMaxPlanes];
  CUtensorMap lo_maps_c1[kHeadMaxPlanes];
};

// Launch the fold program (ns steps, ops/affs/relus as pw_as_fold returns them) + head GEMV when it
// fits this kernel (C in {64, 96, 128}, nb in {2,4,6,8}); returns the kernel name, or nullptr if the caller
// must use another kernel.
const char* launch_head_tma(const PwProgram& prog, int ns, const int* ops, const int* affs, const int* relus,
                            const PlaneGeom& geo, cudaStream_t s);

}  // namespace cnrx
