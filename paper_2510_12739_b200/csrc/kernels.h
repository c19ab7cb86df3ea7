// kernels.h — host-side launchers of the non-GEMM kernels (featurize, pointwise programs / head,
// generic fp32 node kernels).  Every launcher enqueues on the given stream and returns the kernel's
// name (recorded per forward for profiling and for the driver's native-code evidence).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.h"

namespace cnrx {

constexpr int kMaxPilotSyms = 8;

// Interpolation tables for the LS estimate, precomputed once per plan from the pilot grid.
struct PilotTablesDev {
  int32_t n_sym;
  int32_t sym[kMaxPilotSyms];   // pilot symbol indices (ascending)
  const int32_t* flo;           // [n_sym][F] bracketing pilot subcarriers
  const int32_t* fhi;
  const float* wf;              // [n_sym][F] weight of fhi
  const int32_t* jlo;           // [T] bracketing pilot symbols (index into sym)
  const int32_t* jhi;
  const float* wt;              // [T]
  const float* x;               // [T][F] complex pilot grid (0 off-pilot)
  const float* inv_x;           // [T][F] complex 1/x at pilot REs
};

// plane: 16-bit feature plane [Nalloc][cpad], bf16 or (fp16) fp16
const char* launch_featurize_plane(const float* y, const PlaneGeom& geo, int N, const PilotTablesDev& pt,
                                   __nv_bfloat16* plane, int cpad, bool fp16, cudaStream_t s);
// Classical receiver (classic.cu): LMMSE combining + exact max-log demapping per RE.  Either feat
// ([B,T,F,6N] featurizer output: y and the LS-interpolated estimate) or y and h ([B,T,F,N] complex).
const char* launch_lmmse_demap(const float* feat, const float2* y, const float2* h, const float* noise_var, int64_t B,
                               int T, int F, int N, int bits, float* llr, cudaStream_t s);
const char* launch_featurize_ref(const float* y, const PlaneGeom& geo, int N, const PilotTablesDev& pt, float* feat,
                                 cudaStream_t s);
// Test hook: the valid rows of a 16-bit plane [Nalloc][cpad] in reference order [B,T,F,cpad].
const char* launch_plane_rows_to_ref(const __nv_bfloat16* plane, const PlaneGeom& geo, int cpad, uint16_t* out,
                                     cudaStream_t s);
// split: write a split plane [Nalloc][2*cpad] (hi | lo halves, CNRX_*X3 plans)
const char* launch_pack_plane(const float* x, const PlaneGeom& geo, int C, __nv_bfloat16* plane, int cpad, bool fp16,
                              cudaStream_t s, bool split = false);

// ---------------------------------------------------------------------------------------------
// Fused input stage: network input features (computed from the received grid, or read from the
// caller's fp32 [B,T,F,C] tensor) -> every 1x1 "stem" conv on the network input, on CUDA cores
// (12 -> 3 x 64 is 768 FMA per row; a tensor-core launch would be epilogue-bound).
// out = [relu](W . x + bias) (BN folded), optional out2 = relu(out*s2 + t2), padding rows zeroed.
// ---------------------------------------------------------------------------------------------
constexpr int kStemMaxOps = 4, kStemMaxIn = 48;
struct StemOp {
  const float* w;        // [cin][cout] fp32 (reference [1,1,cin,cout], BN scale folded)
  const float* bias;     // [cout]
  __nv_bfloat16* out;    // plane [Nalloc][cout]
  __nv_bfloat16* out2;   // nullable
  const float* s2;       // nullable (out2 = relu(out))
  const float* t2;
  int32_t cout, relu;
};
struct StemLaunch {
  StemOp op[kStemMaxOps];
  int32_t nops, cin;
  int32_t N;             // receive mode: antennas (cin = 6N)
  int32_t mode;          // 0: x fp32 [B,T,F,cin]; 1: received grid y
  int32_t fp16;          // output planes are fp16 (else bf16)
  const float* x;
  const float* y;        // complex [B,T,F,N]
  PilotTablesDev pt;
};
const char* launch_stem(const StemLaunch& L, const PlaneGeom& geo, cudaStream_t s);
bool stem_supported_cin(int cin);

// ---------------------------------------------------------------------------------------------
// Pointwise programs over bf16 planes (fusion nodes, the CoNet interaction and the LLR head).
// A program is a linear chain evaluated per row on an 8-channel accumulator slice:
//   LOAD k: acc = plane[k];  MUL k: acc *= plane[k];  ADD k: acc += plane[k];
//   AFF k: acc = acc*s[k] + t[k] (eval BN);  RELU: acc = max(acc, 0)
// and the result is either stored to a bf16 plane or fed to a 1x1 head GEMV
// (llr[b,t,f,:] = acc . W + bias, fp32, reference layout [B,T,F,bits]).  build_conet's fusion tail
// (network.hpp:534-553: mul -> norm -> mul -> norm ... -> main.out) is exactly such a chain.
// ---------------------------------------------------------------------------------------------
enum PwOp : int32_t { PW_LOAD = 0, PW_AFF = 1, PW_RELU = 2, PW_ADD = 3, PW_MUL = 4 };
constexpr int kPwMaxIns = 24, kPwMaxPlanes = 8, kPwMaxAff = 8, kPwMaxBits = 16;

struct PwIns {
  int32_t op, k;
};

struct PwProgram {
  int32_t n_ins;
  int32_t C;                // channels of every operand (multiple of 8)
  int32_t head_bits;        // 0: store plane; >0: head GEMV with this many outputs
  int32_t n_planes_used;    // planes[0 .. n_planes_used) are operands
  int32_t fp16;             // operand / output planes are fp16 (else bf16)
  int32_t tc_head;          // 64-channel heads may run their GEMV on the tensor core (bf16-rounded z)
  int32_t split;            // split planes (CNRX_*X3 plans): a row is [hi C | lo C], value = hi + lo
  int32_t ln;               // k + 1: the program's result per row is layer-normalised over its channels
                            // (norms.hpp:155-191, double statistics), gain / shift aff_s[k] / aff_t[k]; 0: none
  int32_t ln_c;             // real channel count the statistics run over (<= C)
  PwIns ins[kPwMaxIns];
  const __nv_bfloat16* planes[kPwMaxPlanes];
  const float* aff_s[kPwMaxAff];
  const float* aff_t[kPwMaxAff];
  __nv_bfloat16* out_plane; // [Nalloc][C]
  __nv_bfloat16* out2_plane; // optional relu(out) copy [Nalloc][C] (fold programs only), or null
  const float* head_w;      // [C][head_bits] (reference layout of a 1x1 conv weight)
  const float* head_b;      // [head_bits]
  float* llr;               // [B,T,F,head_bits]
};

const char* launch_pw_program(const PwProgram& prog, const PlaneGeom& geo, cudaStream_t s);
// Depthwise conv (kernels.hpp:197-236) over a plane: per channel, bias then the taps in (dt, df) order in fp32
// (fp32 weights [kh*kw][C]), taps as row offsets of the plane layout (padding rows are zero), the result
// rounded to the plane format (split: hi / lo); padding rows written zero.
const char* launch_dwconv_plane(const __nv_bfloat16* in, __nv_bfloat16* out, const float* w, const float* bias, int C,
                                int kh, int kw, int dil, bool h16, bool split, const PlaneGeom& geo, cudaStream_t s);
// Channel concatenation of two planes (CoNet concat fusion, network.hpp:541-544): out row = [a (ca) | b (cb)]
// (split planes: [a_hi | b_hi | a_lo | b_lo]); ca, cb multiples of 8.
const char* launch_concat_planes(const __nv_bfloat16* a, int ca, const __nv_bfloat16* b, int cb, __nv_bfloat16* out,
                                 bool split, const PlaneGeom& geo, cudaStream_t s);

// Specialised form of the common program shape, a left fold over operand planes:
//   acc = P[0]; [aff_0]; [relu_0];  for i >= 1: acc = acc (mul|add) P[i]; [aff_i]; [relu_i]
// (build_conet's fusion tail).  Returns false if the program is not a fold (caller uses the
// generic interpreter).
bool pw_as_fold(const PwProgram& prog, int* nsteps, int* ops, int* affs, int* relus);

// ---------------------------------------------------------------------------------------------
// Generic fp32 node kernels in the reference layout [B,T,F,C] (CNRX_FP32 plans).
// ---------------------------------------------------------------------------------------------
struct ConvF32 {
  const float* x;       // [B,T,F,cin]
  const float* w;       // [kh,kw,cin,cout]
  const float* bias;    // [cout] or null
  float* y;             // [B,T,F,cout]
  int32_t B, T, F, cin, cout, kh, kw, dil_f;
  // fused epilogue, applied in node order: y = conv+bias; [y = y*s+t]; [relu]; [y = y (op) other]
  const float* aff_s;
  const float* aff_t;
  int32_t relu;
  int32_t other_op;     // 0 none, 6 add, 7 mul (LayerOp values)
  const float* other;
};
const char* launch_conv_f32(const ConvF32& p, cudaStream_t s);

const char* launch_dwconv_f32(const float* x, const float* w, const float* bias, float* y, int B, int T, int F,
                              int C, int kh, int kw, cudaStream_t s);
// y = x*s + t per channel (eval BN, pre-folded exactly like norms.hpp:81-95), optional relu
const char* launch_affine_f32(const float* x, const float* s_, const float* t_, int relu, float* y, int64_t rows,
                              int C, cudaStream_t s);
const char* launch_relu_f32(const float* x, float* y, int64_t n, cudaStream_t s);
const char* launch_binary_f32(int op, const float* a, const float* b, float* y, int64_t n, cudaStream_t s);
const char* launch_layernorm_f32(const float* x, const float* g, const float* b, float* y, int64_t rows, int C,
                                 double eps, cudaStream_t s);
const char* launch_concat_f32(const float* a, int ca, const float* b, int cb, float* y, int64_t rows, cudaStream_t s);

}  // namespace cnrx
