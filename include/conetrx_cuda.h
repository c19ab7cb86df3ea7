/* conetrx_cuda.h — C ABI of the B200-native CoNet-Rx inference engine (libconetrx_cuda.so).
 *
 * Drop-in boundary.  The reference exposes the hot path as a header-only C++ template,
 *     Tensor<T> Network<T>::forward(const Tensor<T>& x, NormMode mode, ForwardCache<T>* cache = nullptr,
 *                                   const std::map<int,T>* overrides = nullptr)
 * (/root/reference/proj/core/include/conetrx/network.hpp:162-163), dispatching the closed LayerOp
 * vocabulary (network.hpp:17) node by node (network.hpp:380-420).  There is no plugin registry, so the
 * replacement takes the network's own description — its GraphNode list (network.hpp:19-26, nodes()
 * :335), NamedParam list (network.hpp:28-33, params() :140) and BN-ready flags (bn_ready() :337) —
 * compiles it once into a device plan, and runs forward on B200.  include/conetrx/gpu_plan.hpp is the
 * C++ wrapper that builds these arrays from a live conetrx::Network<float> and rethrows errors as the
 * reference's exception types; INTEGRATION.md shows the binding.
 *
 * Plain pointers and sizes only; no CUDA, torch or C++ types.  `stream` arguments are cudaStream_t
 * passed as void* (NULL = the plan's own stream).
 */
#ifndef CONETRX_CUDA_H
#define CONETRX_CUDA_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The reference reports errors as exceptions; the C++ wrapper maps them back:
 *   CNRX_ERR_INVALID_ARGUMENT  <- std::invalid_argument from require() (tensor.hpp:13-15), e.g. the
 *                                 channel-count check in forward (network.hpp:164-166)
 *   CNRX_ERR_NOT_READY         <- std::runtime_error for eval-mode BN without statistics (norms.hpp:66-69)
 *   CNRX_ERR_UNSUPPORTED       graph / mode this engine does not run (e.g. NormMode::train, which
 *                              mutates running statistics; no CPU fallback exists by design)
 *   CNRX_ERR_CUDA              a CUDA runtime error (message names the call)                          */
#define CNRX_OK 0
#define CNRX_ERR_INVALID_ARGUMENT 1
#define CNRX_ERR_NOT_READY 2
#define CNRX_ERR_UNSUPPORTED 3
#define CNRX_ERR_CUDA 4

/* LayerOp values (network.hpp:17) */
#define CNRX_OP_INPUT 0
#define CNRX_OP_CONV 1
#define CNRX_OP_DWCONV 2
#define CNRX_OP_RELU 3
#define CNRX_OP_BN 4
#define CNRX_OP_LN 5
#define CNRX_OP_ADD 6
#define CNRX_OP_MUL 7
#define CNRX_OP_CONCAT 8

/* NormMode (norms.hpp:12) */
#define CNRX_MODE_TRAIN 0
#define CNRX_MODE_EVAL 1

/* Arithmetic of the compiled plan.
 *   FP32: CUDA-core fp32 kernels, bit-exact with the reference's float operations.
 *   BF16: bf16 weights/activations with fp32 accumulation on tcgen05 tensor cores (BASELINE's
 *         tensor-core configuration).
 *   FP16: the same tensor-core plan with fp16 weights/activations (11-bit mantissa, |x| <= 65504,
 *         saturating) and an fp32 LLR head: same speed and bytes as BF16, and the mixed-precision
 *         option that meets the >= 99.99 % hard-decision agreement with the reference.
 *   BF16X3: fp32-grade results on the tensor cores (the north star's "LLRs within 1e-4 relative" fp32
 *         path at tensor-core rates): every activation and weight is carried as a 16-bit pair
 *         (hi = bf16(v), lo = bf16(v - hi); 16 significant bits, fp32 range) and each conv is three
 *         tcgen05 products hi*Whi + hi*Wlo + lo*Whi accumulated in fp32; pointwise ops and the head in
 *         fp32.  3x the BF16 plan's tensor work, the bytes of fp32 planes.  Options are fixed (one conv
 *         kernel, separate head).
 *   FP16X3: the same with fp16 pairs (22 significant bits; values must stay within |x| <= 65504). */
#define CNRX_FP32 0
#define CNRX_BF16 1
#define CNRX_FP16 2
#define CNRX_BF16X3 3
#define CNRX_FP16X3 4

/* GraphNode (network.hpp:19-26) + dilation_f (extension for BASELINE config 3; 1 = reference). */
typedef struct {
  int32_t op, in0, in1, w, b, gamma, beta, rmean, rvar, bn_flag, out_channels, dilation_f;
} cnrx_node;

/* NamedParam (network.hpp:28-33): row-major fp32 data, dims[0..rank) (conv weights [kh,kw,Cin,Cout]). */
typedef struct {
  const char* name;
  int32_t rank;
  int32_t learnable;
  int64_t dims[4];
  const float* data;
} cnrx_param;

typedef struct cnrx_plan cnrx_plan;

/* Compile a network into a device plan on `device`.  Validates the graph the way the reference's
 * builders and forward() do; copies (and for BF16 folds/converts) all weights once — the caller's
 * arrays are not referenced afterwards.  Every batch norm must be ready (bn_ready[flag] != 0), as
 * eval-mode forward requires (norms.hpp:66-69). */
int cnrx_plan_create(const cnrx_node* nodes, int32_t n_nodes, int32_t input_node, int32_t output_node,
                     const cnrx_param* params, int32_t n_params, const uint8_t* bn_ready, int32_t n_bn,
                     int32_t precision, int32_t device, cnrx_plan** out);

/* Lowering / execution choices of a plan.  Every choice gives identical LLRs except where noted; they
 * exist for A/B measurements.  cnrx_plan_create uses cnrx_plan_options_default() and then lets the
 * CNRX_* environment variables of DESIGN.md §7 override it (A/B testing only); cnrx_plan_create_ex uses
 * exactly the options passed (NULL = defaults, no environment). */
typedef struct {
  int32_t struct_size;          /* sizeof(cnrx_plan_options): checked for ABI compatibility */
  int32_t fused_blocks;         /* 1: residual blocks of two 64-ch 3x3 convs run as one kernel (default);
                                   0: two weights-stationary conv kernels (env CNRX_BLK=0) */
  int32_t fused_head;           /* 1: the CoNet interaction + LLR head run in the epilogues of the
                                   subnetworks' last convs instead of a separate head kernel (env
                                   CNRX_HEADFUSE=1): on the fused-block program the last blocks run one
                                   launch per subnetwork folding into an fp32 partial plane (LLRs
                                   bit-identical to the head kernel's fp32 GEMV); on the two-kernel
                                   program (BF16 with tensor_core_head) 3-CTA clusters; 0: head kernel */
  int32_t tensor_core_head;     /* 1: 64-ch BF16 heads run their GEMV on the tensor core over bf16-rounded
                                   z (env CNRX_TC_HEAD=1); 0 (default): fp32 CUDA-core GEMV -- one rounding
                                   point fewer; FP16 plans always use fp32 */
  int32_t cta_pair;             /* 1 (default): 96->96 3x3 convs on CTA pairs (cta_group::2); 0: single
                                   CTA (env CNRX_NO_PAIR=1) */
  int32_t weights_stationary;   /* 1 (default): 64->64 3x3 convs with the weights in TMEM; 0: the generic
                                   SS kernel (env CNRX_NO_WS) */
  int32_t relu_on_load;         /* 1 (default): a conv whose input is relu(v) applies it to its shared-
                                   memory window; 0: the producer writes a pre-activated plane
                                   (env CNRX_NO_RELU_IN) */
  int32_t cuda_core_stem;       /* 1: 1x1 stems on the network input run fused with featurize on CUDA
                                   cores in fp32 (env CNRX_STEM=1); 0 (default): tensor-core 1x1 conv --
                                   changes LLRs by the feature / stem-weight rounding */
  int32_t pipeline_chunks;      /* host-buffer entry points: batch chunks overlapping H2D / compute /
                                   D2H; 0 (default) = auto (env CNRX_PIPELINE_CHUNKS) */
  float pipeline_taper;         /* first / last chunk size relative to the others; default 0.125
                                   (env CNRX_PIPELINE_TAPER) */
} cnrx_plan_options;
void cnrx_plan_options_default(cnrx_plan_options* opt);
int cnrx_plan_create_ex(const cnrx_node* nodes, int32_t n_nodes, int32_t input_node, int32_t output_node,
                        const cnrx_param* params, int32_t n_params, const uint8_t* bn_ready, int32_t n_bn,
                        int32_t precision, int32_t device, const cnrx_plan_options* options, cnrx_plan** out);
/* The options a plan was compiled with. */
int cnrx_get_plan_options(const cnrx_plan* plan, cnrx_plan_options* opt);
void cnrx_plan_destroy(cnrx_plan* plan);

/* Thread-local message for the last non-zero status on this thread. */
const char* cnrx_last_error(void);

/* Network<float>::forward(x, mode) (network.hpp:162): x is [B,T,F,C] fp32 channels-last host memory
 * (tensor.hpp:17-19), out receives [B,T,F,output_channels] fp32.  Synchronous.  mode must be
 * CNRX_MODE_EVAL. */
int cnrx_forward(cnrx_plan* plan, const float* x, int64_t B, int64_t T, int64_t F, int64_t C, int32_t mode,
                 float* out);
/* Same with device pointers, enqueued on `stream` (asynchronous). */
int cnrx_forward_device(cnrx_plan* plan, const float* x_dev, int64_t B, int64_t T, int64_t F, int64_t C,
                        int32_t mode, float* out_dev, void* stream);

/* Receiver path (featurize -> subnetworks -> fusion -> head).  The pilot grid is fixed per plan
 * (pilots.cpp:13-31 "identical across samples"): pilots [T,F] complex (re,im) fp32, mask [T,F]. */
int cnrx_set_pilots(cnrx_plan* plan, int64_t T, int64_t F, const float* pilots, const uint8_t* mask);
/* y: [B,T,F,N] complex (re,im) fp32 received grid -> llr [B,T,F,bits] fp32; the plan's input must have
 * 6N channels (per antenna: Re y, Im y, Re x_p, Im x_p, Re h_ls, Im h_ls).  Host memory, synchronous. */
int cnrx_receive(cnrx_plan* plan, const float* y, int64_t B, int64_t T, int64_t F, int64_t N, float* llr);
int cnrx_receive_device(cnrx_plan* plan, const float* y_dev, int64_t B, int64_t T, int64_t F, int64_t N,
                        float* llr_dev, void* stream);
/* Featurize alone (device): feat [B,T,F,6N] fp32 in the reference layout. */
int cnrx_featurize_device(cnrx_plan* plan, const float* y_dev, int64_t B, int64_t T, int64_t F, int64_t N,
                          float* feat_dev, void* stream);

/* Test hook (synchronous): the network-input feature plane exactly as a BF16 / FP16 plan's first
 * convolutions read it -- out_dev receives [B,T,F,cpad] 16-bit values (bf16 or fp16 bits, per the plan;
 * padding channels zero) in the reference order; *cpad = the plan's padded input channel count. */
int cnrx_feature_plane_device(cnrx_plan* plan, const float* y_dev, int64_t B, int64_t T, int64_t F, int64_t N,
                              uint16_t* out_dev, int32_t* cpad);

/* Debug hook: the plan's own bounds check (compute-sanitizer memcheck's stand-in for out-of-range writes).
 * With guard bands on, every workspace allocation of the plan (activation planes, fp32 node buffers,
 * staging, feature and fold buffers) sits between two 256 KB canary bands; cnrx_plan_check_guard_bands
 * synchronises the device and counts canary bytes that no longer hold their pattern (0 = no kernel wrote
 * outside its buffers since they were allocated).  Switching the mode frees the workspace (the next call
 * reallocates it).  No reference counterpart: the reference allocates one Tensor per node
 * (network.hpp:170-178) and relies on the host sanitizers. */
int cnrx_plan_set_guard_bands(cnrx_plan* plan, int32_t enable);
int cnrx_plan_check_guard_bands(cnrx_plan* plan, int64_t* n_buffers, int64_t* bad_bytes);
/* Device address of guard band `side` (0 below, 1 above) of guarded buffer `index` (256 KB each): lets a
 * test of the check itself overwrite a canary. */
int cnrx_plan_guard_band_ptr(cnrx_plan* plan, int64_t index, int32_t side, void** band_dev);

/* Slot-sharded forward / receive across several plans (one per GPU, built from the same network): slots are
 * split into contiguous ranges, each GPU runs its range from host memory on its own thread, LLRs land
 * in the caller's buffer.  No collective on the data path. */
int cnrx_forward_sharded(cnrx_plan* const* plans, int32_t n_plans, const float* x, int64_t B, int64_t T,
                         int64_t F, int64_t C, int32_t mode, float* out);
int cnrx_receive_sharded(cnrx_plan* const* plans, int32_t n_plans, const float* y, int64_t B, int64_t T,
                         int64_t F, int64_t N, float* llr);

/* Introspection for benchmarks and tests. */
typedef struct {
  int32_t precision;
  int32_t device;
  int32_t n_launches;        /* kernels per forward at the last shape (0 before the first forward) */
  int32_t n_tc_convs;        /* convs lowered to tcgen05 implicit GEMM */
  int32_t input_channels;
  int32_t output_channels;
  int64_t macs_per_re;       /* algorithmic MACs per resource element (all taps) */
  int64_t rows_per_slot;     /* padded activation rows per slot in the BF16 plane layout */
  int64_t workspace_bytes;
} cnrx_plan_info;
int cnrx_get_plan_info(const cnrx_plan* plan, cnrx_plan_info* info);

/* Capture the forward of the current shape into a CUDA graph and replay it on subsequent calls
 * with identical (B,T,F) and pointers (enable=1), or disable (0). */
int cnrx_set_graph_capture(cnrx_plan* plan, int32_t enable);

/* Per-launch device timing: with profiling enabled every forward records a CUDA event after each
 * kernel on the launching stream; cnrx_read_profile synchronises, accumulates the per-position
 * durations (ms) and call counts since the last read into ms[]/counts[] (up to max_n entries) and
 * returns the number of positions in *n_out.  Position i is the kernel cnrx_launch_name(i). */
int cnrx_set_profiling(cnrx_plan* plan, int32_t enable);
int cnrx_read_profile(cnrx_plan* plan, int32_t max_n, float* ms, int32_t* counts, int32_t* n_out);

/* Name of the kernel launched at position i of the last forward (for profiling / tests), and its
 * algorithmic FLOPs per resource element (2 x MACs over all taps; 0 for non-GEMM kernels, -1 past
 * the end). */
const char* cnrx_launch_name(const cnrx_plan* plan, int32_t i);
int64_t cnrx_launch_flops(const cnrx_plan* plan, int32_t i);

/* ---------------------------------------------------------------------------------------------
 * On-GPU synthetic slots and BER.  The reference's slot model (SPEC.md:212-220
 * generate_tti, qam.cpp:10-52, pilots.cpp:13-31, TDL/Jakes channel.cpp:37-111, AWGN, optional
 * co-channel QPSK interferer) with Philox4x32-10 random draws addressed by (index, purpose, slot) under
 * `seed`, so any slot range is reproducible independently (slot numbers slot0 .. slot0+B-1).
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t T, F, N;
  int32_t mod_order;          /* 4, 16 or 64 (Gray, qam.cpp:42-52) */
  int32_t n_taps;
  int32_t pilot_spacing;      /* pilot every `spacing`-th subcarrier on the pilot symbols */
  int32_t n_pilot_symbols;    /* <= 8 */
  int32_t has_interferer;     /* config 3: QPSK interferer through an independent channel */
  int32_t pilot_symbols[8];
  double rms_delay_s;         /* 0: exponential PDP e^{-l} over the taps */
  double tap_spacing_s;       /* 0: rms/3, or 1/(F scs) when rms is 0 */
  double doppler_max_hz;      /* per-slot Doppler ~ U[0, max] */
  double scs_hz;
  double cp_fraction;
  double snr_db_lo, snr_db_hi;
  double sir_db_lo, sir_db_hi;
} cnrx_link;

/* y_dev: [B,T,F,N] complex (re,im) fp32; bits_dev: [B,T,F,bits] u8 (0 on pilot REs); h_dev (nullable):
 * [B,T,F,N] complex user channel.  Asynchronous on `stream` (NULL: the legacy default stream). */
int cnrx_generate_slots(const cnrx_link* link, int64_t B, uint64_t seed, uint64_t slot0, float* y_dev,
                        uint8_t* bits_dev, float* h_dev, void* stream);
/* Per-slot hard-decision bit errors (LLR > 0 => bit 1) over data REs (data_mask_dev [T,F]
 * u8, 1 = data; pilots excluded): errors_dev [B] u64.  Asynchronous on `stream`. */
int cnrx_count_bit_errors(const float* llr_dev, const uint8_t* bits_dev, const uint8_t* data_mask_dev, int64_t B,
                          int64_t T, int64_t F, int32_t bits, unsigned long long* errors_dev, void* stream);

/* Per-slot total noise-plus-interference variance of the generated slots (interference as noise:
 * 10^(-SNR/10) + 10^(-SIR/10) with the interferer's unit-power channel), host output [B]. */
int cnrx_slot_noise_var(const cnrx_link* link, int64_t B, uint64_t seed, uint64_t slot0, float* noise_var);

/* Classical baseline receiver: LMMSE combining over the N
 * antennas + exact max-log demapping (Gray QAM, positive LLR => bit 1).  h_dev == NULL: LS estimate with
 * the plan's pilot grid and the featurizer's interpolation (ls_lmmse); otherwise h_dev [B,T,F,N] complex
 * is the true channel (perfect_csi_lmmse).  noise_var_dev [B]: total noise(+interference) variance.
 * llr_dev [B,T,F,bits] fp32.  Asynchronous on `stream` (NULL: the plan's stream). */
int cnrx_classical_receive(cnrx_plan* plan, const float* y_dev, const float* h_dev, const float* noise_var_dev,
                           int64_t B, int64_t T, int64_t F, int64_t N, int32_t mod_order, float* llr_dev,
                           void* stream);

/* Peer-memory LLR gather (one process per GPU, the final LLR gather fused into the last
 * kernel).  Rank 0 allocates the whole batch's LLR buffer with cnrx_ipc_alloc and shares the 64-byte
 * CUDA IPC handle; every rank opens it (cnrx_ipc_open) and passes base + (its first slot) * T*F*bits as
 * the llr_dev of cnrx_receive_device / cnrx_forward_device: the LLR head's stores then land directly in
 * rank 0's HBM over NVLink -- no gather collective, no staging copy.  Completion: each rank synchronizes
 * its stream, then a host barrier; rank 0 then owns the full batch. */
typedef struct {
  uint8_t bytes[64];
} cnrx_ipc_handle;
int cnrx_ipc_alloc(int32_t device, int64_t bytes, void** ptr_out, cnrx_ipc_handle* handle_out);
int cnrx_ipc_open(int32_t device, const cnrx_ipc_handle* handle, void** ptr_out);
int cnrx_ipc_close(int32_t device, void* opened_ptr);
int cnrx_ipc_free(int32_t device, void* allocated_ptr);
/* Synchronous copy of `bytes` from a (local or opened) device buffer to host memory. */
int cnrx_ipc_read(int32_t device, const void* src, void* host_dst, int64_t bytes);
/* The same copy enqueued on `stream` (a cudaStream_t of `device`; host_dst pinned), not waited for: rank 0
 * reads step k's batch on a side stream while step k + 1 computes into the other buffer of a pair. */
int cnrx_ipc_read_async(int32_t device, const void* src, void* host_dst, int64_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CONETRX_CUDA_H */
