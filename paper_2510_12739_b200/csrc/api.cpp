// api.cpp — the C ABI (include/conetrx_cuda.h): plan creation, the plan compiler and the executor.
//
// A plan is compiled once from the reference network's own description (GraphNode list + named
// params + BN-ready flags, network.hpp:19-33,335-337) and then runs Network<float>::forward
// (network.hpp:162-180) on the GPU:
//
//   CNRX_FP32  node-level executor in the reference layout [B,T,F,C]: every LayerOp has an fp32 CUDA
//              kernel (generic_f32.cu); a conv absorbs the single-consumer BN / ReLU / add|mul chain
//              after it.  Any graph the reference builders produce runs on this path.
//   CNRX_BF16  lowering onto tcgen05 implicit-GEMM convolutions over bf16 activation planes
//   CNRX_FP16  (the same lowering over fp16 planes / weights, fp32 LLR head; everything below that says
//              "bf16 plan" applies to both 16-bit formats)
//              (conv_tc.cu): BN after a conv is folded into its weights, ReLU / residual add / the next
//              block's pre-activation go into the conv epilogue, same-level convs of different
//              subnetworks share one grouped launch, and the fusion tail + 1x1 head is a single
//              pointwise-program kernel (pointwise.cu).  Graph shapes the lowering cannot express are
//              rejected with CNRX_ERR_UNSUPPORTED — there is no CPU fallback anywhere.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/conetrx_cuda.h"
#include "common.h"
#include "conv_tc.h"
#include "conv_x3.h"
#include "conv_blk.h"
#include "conv_pair.h"
#include "conv_ws.h"
#include "slotgen.h"
#include "kernels.h"


namespace cnrx {
void ensure_smem_attr(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  CNRX_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  int& have = done[{dev, func}];
  if (have >= bytes) return;
  CNRX_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CNRX_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared));
  have = bytes;
}
}  // namespace cnrx

using namespace cnrx;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return CNRX_OK;
  } catch (const Error& e) {
    return fail(e.code, e.what());
  } catch (const std::exception& e) {
    return fail(CNRX_ERR_INVALID_ARGUMENT, e.what());
  }
}

struct HostParam {
  std::string name;
  std::vector<int64_t> dims;
  std::vector<float> data;
  bool learnable = true;
  int64_t numel() const {
    int64_t n = 1;
    for (auto d : dims) n *= d;
    return n;
  }
};

constexpr double kBnEps = 1e-5;  // network.hpp:429
constexpr double kLnEps = 1e-5;  // network.hpp:431

// Eval BN as a per-channel affine, computed exactly like norms.hpp:81-88 (istd in double, then float).
void bn_affine(const HostParam& g, const HostParam& s, const HostParam& rm, const HostParam& rv,
               std::vector<float>& scale, std::vector<float>& shift) {
  const size_t c = g.data.size();
  scale.resize(c);
  shift.resize(c);
  for (size_t i = 0; i < c; ++i) {
    const float istd = static_cast<float>(1.0 / std::sqrt(static_cast<double>(rv.data[i]) + kBnEps));
    scale[i] = g.data[i] * istd;
    shift[i] = s.data[i] - rm.data[i] * scale[i];
  }
}

int round_cin(int c) {
  if (c <= 16) return 16;
  if (c <= 32) return 32;
  if (c <= 64) return 64;
  if (c <= 96) return 96;
  return (c + 63) / 64 * 64;
}
int round_cout(int c) { return (c + 31) / 32 * 32; }

// ------------------------------------------------------------------------------------------------
// FP32 program
// ------------------------------------------------------------------------------------------------
enum F32Kind { F_CONV, F_DWCONV, F_AFFINE, F_RELU, F_BINARY, F_LN, F_CONCAT };
struct F32Step {
  F32Kind kind;
  int out_val;              // value id written
  int in0 = -1, in1 = -1;   // value ids read
  int node = -1;            // primary node
  ConvF32 conv{};           // static parts (weights, epilogue tables)
  int op = 0;               // binary op
  int relu = 0;
  const float* s = nullptr;
  const float* t = nullptr;
  const float* g = nullptr;
  const float* b = nullptr;
  int C = 0, C2 = 0, kh = 0, kw = 0;
  const float* w = nullptr;
  const float* bias = nullptr;
};

// ------------------------------------------------------------------------------------------------
// BF16 program
// ------------------------------------------------------------------------------------------------
struct PlaneInfo {
  int C = 0;           // padded channels
  bool nonneg = false; // every valid value >= 0 (output of a ReLU)
  int level = 0;       // level of its producer
  int last_use = 0;    // last level reading it
  int buffer = -1;     // workspace buffer index
};
struct TcOp {
  int node = -1;
  int cin = 0, cout = 0, ks = 1, dil = 1;
  int cin_real = 0, cout_real = 0;
  bool ws = false;  // weights-stationary (A in TMEM) 64->64 3x3 kernel
  bool stem = false;             // 1x1 conv on the network input, run by the fused stem kernel
  float* stem_w = nullptr;       // fp32 [cin_real][cout_real], BN scale folded
  int in_plane = -1, res_plane = -1, out_plane = -1, out2_plane = -1;
  int relu = 0;
  int relu_in = 0;  // ws kernels: input is relu(in_plane), applied to the window on load
  // fused residual block (conv_blk.cu): this op is conv2 and `blk_c1` its conv1 (`fused_away`).  When
  // the workspace runs blocks fused, conv1 is not launched and its output plane is not written; the
  // two-kernel program over the same planes stays available (chosen per batch size).
  int blk_c1 = -1;
  bool fused_away = false;
  bool llr_head = false;  // the network's output conv (3x3 head): its epilogue writes the fp32 LLRs
  void* wimg = nullptr;
  float* bias = nullptr;
  float* s2 = nullptr;
  float* t2 = nullptr;
  int level = 0;
};
struct PwStep {
  PwProgram prog{};
  bool concat = false;  // channel concatenation of plane_ids[0], plane_ids[1] (launch_concat_planes)
  bool dw = false;      // depthwise conv of plane_ids[0] (launch_dwconv_plane)
  const float* dw_w = nullptr;
  const float* dw_b = nullptr;
  int dw_kh = 0, dw_kw = 0, dw_dil = 1;
  int plane_ids[kPwMaxPlanes];
  int n_planes = 0;
  int out_plane = -1;  // -1: head
  int out2_plane = -1; // relu(out) copy (fold programs): the next block's pre-activation
  int level = 0;
};

struct Workspace {
  int B = -1, T = -1, F = -1;
  int cap_B = 0;  // batch the buffers were allocated for
  PlaneGeom geo{};
  std::vector<void*> buffers;
  std::vector<size_t> sizes;
  void* in_buf = nullptr;   // device copy of host input
  size_t in_bytes = 0;
  void* out_buf = nullptr;  // device output for host APIs
  size_t out_bytes = 0;
  void* feat_buf = nullptr; // fp32 features when an FP32 plan runs the receive path
  size_t feat_bytes = 0;
  void* classic_buf = nullptr;  // fp32 features of the classical LS-LMMSE receiver
  size_t classic_bytes = 0;
  struct GroupLaunch {
    bool ws = false;
    bool blk = false;
    bool skip = false;  // conv1 group of fused blocks while the workspace runs them fused
    bool pair = false;  // conv_pair.cu (CTA-pair 96 -> 96 3x3)
    bool x3 = false;    // conv_x3.cu (split-precision plans)
    TcLaunch tc;
    X3Launch x3l;
    WsLaunch wsl;
    BlkLaunch blkl;
    std::vector<BlkLaunch> chain;  // fused-block head: one block launch per subnetwork, in fold order
  };
  std::vector<GroupLaunch> launches;  // prepared tensor maps per TC group (bf16)
  bool blocks_fused = false;          // residual blocks run as conv_blk64 at this batch size
  bool head_fused = false;            // the head runs in the last convs' epilogue (two-kernel program)
  bool head_blk_fused = false;        // ... in the last fused blocks' conv2 epilogues (fused-block program)
  void* fold_bufs[2] = {nullptr, nullptr};  // fp32 partial-fold planes [Nalloc][64] of the fused-block head
  size_t fold_bytes = 0;
  // guard bands (cnrx_plan_set_guard_bands): every workspace allocation sits between two canary bands
  bool guard = false;
  struct Guarded {
    char* base;
    size_t bytes;
  };
  std::vector<Guarded> guarded;
};

constexpr size_t kGuardBytes = 256u << 10;  // > one TMA window / staged tile either side; keeps 1 KB alignment
constexpr int kGuardByte = 0xA5;

// Workspace allocations go through these two, so a plan in guard-band mode can check that no kernel
// wrote outside its buffers (the pool's compute-sanitizer is closed; this is the plan's own bounds check).
void* ws_malloc(Workspace& ws, size_t bytes) {
  void* d = nullptr;
  if (!ws.guard) {
    CNRX_CUDA(cudaMalloc(&d, bytes));
    return d;
  }
  CNRX_CUDA(cudaMalloc(&d, bytes + 2 * kGuardBytes));
  char* base = static_cast<char*>(d);
  cudaError_t e = cudaMemset(base, kGuardByte, kGuardBytes);
  if (e == cudaSuccess) e = cudaMemset(base + kGuardBytes + bytes, kGuardByte, kGuardBytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // the memsets run on the legacy stream, forwards do not
  if (e != cudaSuccess) {
    cudaFree(base);
    CNRX_CUDA(e);
  }
  ws.guarded.push_back({base, bytes});
  return base + kGuardBytes;
}

void ws_free(Workspace& ws, void* ptr) {
  if (!ptr) return;
  for (size_t i = 0; i < ws.guarded.size(); ++i)
    if (ws.guarded[i].base + kGuardBytes == ptr) {
      cudaFree(ws.guarded[i].base);
      ws.guarded.erase(ws.guarded.begin() + static_cast<std::ptrdiff_t>(i));
      return;
    }
  cudaFree(ptr);
}

}  // namespace

struct cnrx_plan {
  int precision = CNRX_FP32;
  bool fp16 = false;           // CNRX_FP16 / CNRX_FP16X3: the 16-bit planes and weights are fp16
  bool split = false;          // CNRX_BF16X3 / CNRX_FP16X3: planes and weights carried as (hi, lo) pairs
  cnrx_plan_options opt{};
  int device = 0;
  int num_sms = 148;
  size_t mem_budget = 0;       // workspace bytes one forward may use; larger batches run in slot chunks
  cudaStream_t stream = nullptr;
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the pipelined host APIs
  std::vector<cudaEvent_t> pipe_ev;            // [2 * chunks]: input landed / chunk computed
  std::vector<cnrx_node> nodes;
  int in_node = -1, out_node = -1;
  std::vector<HostParam> params;
  std::vector<uint8_t> bn_ready;
  std::vector<std::vector<int>> consumers;
  int in_ch = 0, out_ch = 0;
  int64_t macs = 0;
  std::vector<void*> dev_allocs;

  // fp32
  std::vector<F32Step> f32;
  std::vector<int> f32_val_channels;  // channels of each value
  std::vector<int> f32_val_buffer;    // buffer index per value (-1 = external input/output)
  int f32_in_val = -1, f32_out_val = -1;
  int f32_nbuf = 0;
  std::vector<int> f32_buf_channels;

  // bf16
  std::vector<PlaneInfo> planes;
  std::vector<TcOp> tc;
  std::vector<PwStep> pw;
  std::vector<std::vector<std::vector<int>>> tc_groups_by_level;  // [level] -> groups -> op ids
  std::vector<std::vector<int>> pw_by_level;
  int n_levels = 0;
  int npad = 1;
  std::vector<int> stem_ops;   // TcOp indices run by the fused stem kernel
  // fused interaction + LLR head (conv_ws.cu kWsHead): the tc group (level, index) whose convs produce
  // every operand of the head's fold, in fold order, and the head's pointwise step it replaces
  int hf_level = -1, hf_group = -1, hf_pw = -1;
  // interaction + head folded into the last fused blocks (conv_blk.cu BlkFold): the tc group (level, index)
  // of those blocks, its ops in fold order, the head's pointwise step, and the fold steps
  int hb_level = -1, hb_group = -1, hb_pw = -1, hb_ns = 0;
  int hb_ops[kPwMaxPlanes] = {}, hb_affs[kPwMaxPlanes] = {}, hb_relus[kPwMaxPlanes] = {}, hb_tc[kPwMaxPlanes] = {};
  WsHead hf{};
  bool need_plane0 = true;     // some kernel reads the input-feature plane
  std::vector<int> buf_channels;  // plane buffers

  // pilots
  bool has_pilots = false;
  int pT = 0, pF = 0;
  PilotTablesDev pt{};

  Workspace ws;
  std::vector<std::string> launch_names;
  std::mutex mu;

  // per-launch profiling (events around every launch of a forward)
  bool profile = false;
  std::vector<std::vector<cudaEvent_t>> prof_events;  // one vector per profiled forward
  std::vector<cudaEvent_t> event_pool;
  std::vector<double> prof_ms;
  std::vector<int32_t> prof_count;
  cudaEvent_t take_event() {
    cudaEvent_t e;
    if (!event_pool.empty()) {
      e = event_pool.back();
      event_pool.pop_back();
    } else {
      CNRX_CUDA(cudaEventCreate(&e));
    }
    return e;
  }
  std::vector<int64_t> launch_flops;  // algorithmic FLOP per resource element of each launch
  void note(const char* name, cudaStream_t s, int64_t flops_per_re = 0) {
    launch_names.emplace_back(name);
    launch_flops.push_back(flops_per_re);
    if (profile && !prof_events.empty()) {
      cudaEvent_t e = take_event();
      CNRX_CUDA(cudaEventRecord(e, s));
      prof_events.back().push_back(e);
    }
  }

  // graph capture
  bool capture = false;
  cudaEvent_t fence_in = nullptr, fence_out = nullptr;
  cudaEvent_t ws_done = nullptr;       // end of the last forward's work on the shared workspace
  cudaStream_t ws_stream = nullptr;    // stream that forward ran on
  bool ws_used = false;
  cudaEvent_t classic_done = nullptr;  // end of the last classical receive on classic_buf
  cudaStream_t classic_stream = nullptr;
  bool classic_used = false;
  cudaGraphExec_t gexec = nullptr;
  std::string gkey;

  float* upload(const std::vector<float>& v) {
    float* d = nullptr;
    CNRX_CUDA(cudaMalloc(&d, std::max<size_t>(1, v.size()) * sizeof(float)));
    dev_allocs.push_back(d);
    if (!v.empty()) CNRX_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice));
    return d;
  }
  void* upload_bytes(const void* p, size_t n) {
    void* d = nullptr;
    CNRX_CUDA(cudaMalloc(&d, std::max<size_t>(16, n)));
    dev_allocs.push_back(d);
    CNRX_CUDA(cudaMemcpy(d, p, n, cudaMemcpyHostToDevice));
    return d;
  }
  const HostParam& P(int i) const { return params[static_cast<size_t>(i)]; }
  const cnrx_node& N(int i) const { return nodes[static_cast<size_t>(i)]; }
  int single_consumer(int i) const {
    const auto& c = consumers[static_cast<size_t>(i)];
    return c.size() == 1 ? c[0] : -1;
  }
};

namespace {

// ------------------------------------------------------------------------------------------------
// Validation (mirrors the checks the reference's builders and forward perform)
// ------------------------------------------------------------------------------------------------
void validate_graph(cnrx_plan& p) {
  const int n = static_cast<int>(p.nodes.size());
  require(p.in_node >= 0 && p.in_node < n && p.out_node >= 0 && p.out_node < n, "network has no input/output");
  require(p.N(p.in_node).op == CNRX_OP_INPUT, "input node is not an input op");
  p.consumers.assign(static_cast<size_t>(n), {});
  auto param_ok = [&](int idx) { return idx >= 0 && idx < static_cast<int>(p.params.size()); };
  for (int i = 0; i < n; ++i) {
    const cnrx_node& nd = p.N(i);
    if (nd.op == CNRX_OP_INPUT) {
      require(i == p.in_node, "network already has an input node");
      continue;
    }
    require(nd.in0 >= 0 && nd.in0 < i, "bad input node index");
    const int cin = p.N(nd.in0).out_channels;
    if (nd.in1 >= 0) require(nd.in1 < i, "bad input node index");
    p.consumers[static_cast<size_t>(nd.in0)].push_back(i);
    if (nd.in1 >= 0) p.consumers[static_cast<size_t>(nd.in1)].push_back(i);
    switch (nd.op) {
      case CNRX_OP_CONV: {
        require(param_ok(nd.w), "conv without weights");
        const auto& w = p.P(nd.w);
        require(w.dims.size() == 4, "conv weights must be [kh,kw,Cin,Cout]");
        require(w.dims[0] % 2 == 1 && w.dims[1] % 2 == 1, "conv kernel dims must be odd");
        require(w.dims[2] == cin, "conv input has " + std::to_string(cin) + " channels but weights expect " +
                                      std::to_string(w.dims[2]));
        require(w.dims[3] == nd.out_channels, "conv output channel mismatch");
        if (nd.b >= 0) require(param_ok(nd.b) && p.P(nd.b).numel() == w.dims[3], "conv bias must be [Cout]");
        require(nd.dilation_f >= 1, "dilation must be >= 1");
        p.macs += w.dims[0] * w.dims[1] * w.dims[2] * w.dims[3];
        break;
      }
      case CNRX_OP_DWCONV: {
        require(param_ok(nd.w), "dwconv without weights");
        const auto& w = p.P(nd.w);
        require(w.dims.size() == 4 && w.dims[3] == 1 && w.dims[2] == cin, "depthwise weights must be [kh,kw,C,1]");
        p.macs += w.dims[0] * w.dims[1] * w.dims[2];
        break;
      }
      case CNRX_OP_BN:
        require(param_ok(nd.gamma) && param_ok(nd.beta) && param_ok(nd.rmean) && param_ok(nd.rvar),
                "batch norm parameters missing");
        require(p.P(nd.gamma).numel() == cin && p.P(nd.beta).numel() == cin && p.P(nd.rmean).numel() == cin &&
                    p.P(nd.rvar).numel() == cin,
                "batch norm gain must be [C]");
        require(nd.bn_flag >= 0 && nd.bn_flag < static_cast<int>(p.bn_ready.size()), "bad bn flag");
        if (!p.bn_ready[static_cast<size_t>(nd.bn_flag)])
          throw Error(CNRX_ERR_NOT_READY,
                      "batch norm evaluated in eval mode before any train-mode update; train first or seed the "
                      "running statistics");
        break;
      case CNRX_OP_LN:
        require(param_ok(nd.gamma) && param_ok(nd.beta) && p.P(nd.gamma).numel() == cin && p.P(nd.beta).numel() == cin,
                "layer norm gain must be [C]");
        break;
      case CNRX_OP_ADD:
      case CNRX_OP_MUL:
        require(nd.in1 >= 0, "binary op needs two inputs");
        require(p.N(nd.in1).out_channels == cin, "elementwise fusion requires equal channel counts");
        break;
      case CNRX_OP_CONCAT:
        require(nd.in1 >= 0, "concat needs two inputs");
        require(nd.out_channels == cin + p.N(nd.in1).out_channels, "concat output channel mismatch");
        break;
      case CNRX_OP_RELU:
        break;
      default:
        throw Error(CNRX_ERR_INVALID_ARGUMENT, "unknown op " + std::to_string(nd.op));
    }
    // shape-preserving ops: every buffer is sized from out_channels, so it must equal the input's
    if (nd.op == CNRX_OP_RELU || nd.op == CNRX_OP_BN || nd.op == CNRX_OP_LN || nd.op == CNRX_OP_ADD ||
        nd.op == CNRX_OP_MUL || nd.op == CNRX_OP_DWCONV)
      require(nd.out_channels == cin, "node " + std::to_string(i) + ": output channels must equal its input's");
  }
  p.in_ch = p.N(p.in_node).out_channels;
  p.out_ch = p.N(p.out_node).out_channels;
  for (auto& nd : p.nodes)
    p.npad = std::max(p.npad, nd.op == CNRX_OP_CONV || nd.op == CNRX_OP_DWCONV ? nd.dilation_f : 1);
}

// ------------------------------------------------------------------------------------------------
// FP32 compile
// ------------------------------------------------------------------------------------------------
void compile_f32(cnrx_plan& p) {
  const int n = static_cast<int>(p.nodes.size());
  std::vector<int> val_of(static_cast<size_t>(n), -1);
  std::vector<char> absorbed(static_cast<size_t>(n), 0);
  auto new_val = [&](int C) {
    p.f32_val_channels.push_back(C);
    return static_cast<int>(p.f32_val_channels.size()) - 1;
  };
  p.f32_in_val = new_val(p.in_ch);
  val_of[static_cast<size_t>(p.in_node)] = p.f32_in_val;
  for (int i = 0; i < n; ++i) {
    if (i == p.in_node || absorbed[static_cast<size_t>(i)]) continue;
    const cnrx_node& nd = p.N(i);
    F32Step st{};
    st.node = i;
    st.in0 = val_of[static_cast<size_t>(nd.in0)];
    int end = i;
    switch (nd.op) {
      case CNRX_OP_CONV: {
        st.kind = F_CONV;
        const auto& w = p.P(nd.w);
        st.conv.w = p.upload(w.data);
        st.conv.bias = nd.b >= 0 ? p.upload(p.P(nd.b).data) : nullptr;
        st.conv.kh = static_cast<int>(w.dims[0]);
        st.conv.kw = static_cast<int>(w.dims[1]);
        st.conv.cin = static_cast<int>(w.dims[2]);
        st.conv.cout = static_cast<int>(w.dims[3]);
        st.conv.dil_f = nd.dilation_f;
        int c = p.single_consumer(end);
        if (c >= 0 && p.N(c).op == CNRX_OP_BN && end != p.out_node) {
          std::vector<float> s, t;
          const auto& bn = p.N(c);
          bn_affine(p.P(bn.gamma), p.P(bn.beta), p.P(bn.rmean), p.P(bn.rvar), s, t);
          st.conv.aff_s = p.upload(s);
          st.conv.aff_t = p.upload(t);
          absorbed[static_cast<size_t>(c)] = 1;
          end = c;
          c = p.single_consumer(end);
        }
        if (c >= 0 && p.N(c).op == CNRX_OP_RELU && end != p.out_node) {
          st.conv.relu = 1;
          absorbed[static_cast<size_t>(c)] = 1;
          end = c;
          c = p.single_consumer(end);
        }
        if (c >= 0 && (p.N(c).op == CNRX_OP_ADD || p.N(c).op == CNRX_OP_MUL) && end != p.out_node) {
          const int other = p.N(c).in0 == end ? p.N(c).in1 : p.N(c).in0;
          if (other != end && other < i && val_of[static_cast<size_t>(other)] >= 0) {
            st.conv.other_op = p.N(c).op;
            st.in1 = val_of[static_cast<size_t>(other)];
            absorbed[static_cast<size_t>(c)] = 1;
            end = c;
          }
        }
        break;
      }
      case CNRX_OP_DWCONV: {
        st.kind = F_DWCONV;
        const auto& w = p.P(nd.w);
        st.w = p.upload(w.data);
        st.bias = nd.b >= 0 ? p.upload(p.P(nd.b).data) : nullptr;
        st.kh = static_cast<int>(w.dims[0]);
        st.kw = static_cast<int>(w.dims[1]);
        break;
      }
      case CNRX_OP_BN: {
        st.kind = F_AFFINE;
        std::vector<float> s, t;
        bn_affine(p.P(nd.gamma), p.P(nd.beta), p.P(nd.rmean), p.P(nd.rvar), s, t);
        st.s = p.upload(s);
        st.t = p.upload(t);
        const int c = p.single_consumer(i);
        if (c >= 0 && p.N(c).op == CNRX_OP_RELU && i != p.out_node) {
          st.relu = 1;
          absorbed[static_cast<size_t>(c)] = 1;
          end = c;
        }
        break;
      }
      case CNRX_OP_RELU:
        st.kind = F_RELU;
        break;
      case CNRX_OP_ADD:
      case CNRX_OP_MUL:
        st.kind = F_BINARY;
        st.op = nd.op;
        st.in1 = val_of[static_cast<size_t>(nd.in1)];
        break;
      case CNRX_OP_LN:
        st.kind = F_LN;
        st.g = p.upload(p.P(nd.gamma).data);
        st.b = p.upload(p.P(nd.beta).data);
        break;
      case CNRX_OP_CONCAT:
        st.kind = F_CONCAT;
        st.in1 = val_of[static_cast<size_t>(nd.in1)];
        st.C2 = p.N(nd.in1).out_channels;
        break;
      default:
        throw Error(CNRX_ERR_UNSUPPORTED, "op not supported");
    }
    st.C = p.N(nd.in0).out_channels;
    st.out_val = new_val(p.N(end).out_channels);
    val_of[static_cast<size_t>(end)] = st.out_val;
    p.f32.push_back(st);
  }
  p.f32_out_val = val_of[static_cast<size_t>(p.out_node)];
  require(p.f32_out_val >= 0, "output node is not computed");
  // buffer assignment by liveness (values live from their producing step to their last reader)
  const int nv = static_cast<int>(p.f32_val_channels.size());
  std::vector<int> last(static_cast<size_t>(nv), -1);
  for (int s = 0; s < static_cast<int>(p.f32.size()); ++s) {
    const auto& st = p.f32[static_cast<size_t>(s)];
    if (st.in0 >= 0) last[static_cast<size_t>(st.in0)] = s;
    if (st.in1 >= 0) last[static_cast<size_t>(st.in1)] = s;
  }
  p.f32_val_buffer.assign(static_cast<size_t>(nv), -1);
  std::vector<int> free_at;  // per buffer: step after which it is free
  for (int s = 0; s < static_cast<int>(p.f32.size()); ++s) {
    auto& st = p.f32[static_cast<size_t>(s)];
    if (st.out_val == p.f32_out_val) continue;  // external
    const int C = p.f32_val_channels[static_cast<size_t>(st.out_val)];
    int chosen = -1;
    for (int b = 0; b < p.f32_nbuf; ++b)
      if (p.f32_buf_channels[static_cast<size_t>(b)] == C && free_at[static_cast<size_t>(b)] < s) {
        chosen = b;
        break;
      }
    if (chosen < 0) {
      chosen = p.f32_nbuf++;
      p.f32_buf_channels.push_back(C);
      free_at.push_back(0);
    }
    p.f32_val_buffer[static_cast<size_t>(st.out_val)] = chosen;
    free_at[static_cast<size_t>(chosen)] = std::max(s, last[static_cast<size_t>(st.out_val)]);
  }
}

// ------------------------------------------------------------------------------------------------
// BF16 compile
// ------------------------------------------------------------------------------------------------
struct Bf16Compiler {
  cnrx_plan& p;
  std::vector<int> node_plane;    // node -> plane holding its value
  std::vector<int> plane_producer_tc;  // plane -> tc op index that writes it as primary/out2 (-1 none)
  std::vector<int> plane_producer_pw;  // plane -> pointwise step that writes it as primary (-1 none)

  explicit Bf16Compiler(cnrx_plan& pl) : p(pl) {}

  int new_plane(int C, int level, bool nonneg) {
    PlaneInfo pi;
    pi.C = C;
    pi.level = level;
    pi.nonneg = nonneg;
    p.planes.push_back(pi);
    plane_producer_tc.push_back(-1);
    plane_producer_pw.push_back(-1);
    return static_cast<int>(p.planes.size()) - 1;
  }
  void use(int plane, int level) {
    auto& pi = p.planes[static_cast<size_t>(plane)];
    pi.last_use = std::max(pi.last_use, level);
  }

  // Linear pointwise chain ending at node u whose leaves are planes.  Appends instructions and
  // returns true on success.
  bool build_chain(int u, PwStep& st, std::vector<std::vector<float>>& aff_tables, int& level) {
    if (node_plane[static_cast<size_t>(u)] >= 0) {
      const int pl = node_plane[static_cast<size_t>(u)];
      if (st.n_planes >= kPwMaxPlanes) return false;
      st.plane_ids[st.n_planes] = pl;
      st.prog.ins[st.prog.n_ins++] = {PW_LOAD, st.n_planes++};
      level = std::max(level, p.planes[static_cast<size_t>(pl)].level);
      return true;
    }
    const cnrx_node& nd = p.N(u);
    if (st.prog.n_ins >= kPwMaxIns - 1) return false;
    if (nd.op == CNRX_OP_LN) {  // a layer norm is a row-wise program of its own: its plane is a leaf here
      plane_for(u);
      return build_chain(u, st, aff_tables, level);
    }
    switch (nd.op) {
      case CNRX_OP_RELU:
        if (!build_chain(nd.in0, st, aff_tables, level)) return false;
        st.prog.ins[st.prog.n_ins++] = {PW_RELU, 0};
        return true;
      case CNRX_OP_BN: {
        if (!build_chain(nd.in0, st, aff_tables, level)) return false;
        std::vector<float> s, t;
        bn_affine(p.P(nd.gamma), p.P(nd.beta), p.P(nd.rmean), p.P(nd.rvar), s, t);
        const int k = static_cast<int>(aff_tables.size()) / 2;
        if (k >= kPwMaxAff) return false;
        aff_tables.push_back(s);
        aff_tables.push_back(t);
        st.prog.ins[st.prog.n_ins++] = {PW_AFF, k};
        return true;
      }
      case CNRX_OP_ADD:
      case CNRX_OP_MUL: {
        // one operand must be a plane leaf (a layer norm operand becomes one)
        for (int o : {nd.in0, nd.in1})
          if (node_plane[static_cast<size_t>(o)] < 0 && p.N(o).op == CNRX_OP_LN) plane_for(o);
        int leaf = -1, rest = -1;
        if (node_plane[static_cast<size_t>(nd.in1)] >= 0) {
          leaf = nd.in1;
          rest = nd.in0;
        } else if (node_plane[static_cast<size_t>(nd.in0)] >= 0) {
          leaf = nd.in0;
          rest = nd.in1;
        } else {
          return false;
        }
        if (!build_chain(rest, st, aff_tables, level)) return false;
        const int pl = node_plane[static_cast<size_t>(leaf)];
        if (st.n_planes >= kPwMaxPlanes) return false;
        st.plane_ids[st.n_planes] = pl;
        st.prog.ins[st.prog.n_ins++] = {nd.op == CNRX_OP_MUL ? PW_MUL : PW_ADD, st.n_planes++};
        level = std::max(level, p.planes[static_cast<size_t>(pl)].level);
        return true;
      }
      default:
        return false;
    }
  }

  void finish_pw(PwStep& st, std::vector<std::vector<float>>& aff_tables, int C) {
    st.prog.C = C;
    st.prog.n_planes_used = st.n_planes;
    for (size_t k = 0; k < aff_tables.size() / 2; ++k) {
      auto s = aff_tables[2 * k], t = aff_tables[2 * k + 1];
      s.resize(static_cast<size_t>(C), 0.f);
      t.resize(static_cast<size_t>(C), 0.f);
      st.prog.aff_s[k] = p.upload(s);
      st.prog.aff_t[k] = p.upload(t);
    }
    for (int k = 0; k < st.n_planes; ++k) use(st.plane_ids[k], st.level);
  }

  // Materialise node u as a plane (for a conv input or a residual operand).
  int plane_for(int u) {
    int pl = node_plane[static_cast<size_t>(u)];
    if (pl >= 0) return pl;
    const cnrx_node& nd = p.N(u);
    // relu(v) / relu(bn(v)) where v's plane comes from a TC epilogue: second epilogue output.
    if (nd.op == CNRX_OP_RELU) {
      int v = nd.in0;
      const cnrx_node* bn = nullptr;
      if (node_plane[static_cast<size_t>(v)] < 0 && p.N(v).op == CNRX_OP_BN &&
          node_plane[static_cast<size_t>(p.N(v).in0)] >= 0) {
        bn = &p.N(v);
        v = p.N(v).in0;
      }
      const int vp = node_plane[static_cast<size_t>(v)];
      if (vp >= 0) {
        if (!bn && p.planes[static_cast<size_t>(vp)].nonneg) {  // relu(relu(x)) = relu(x)
          node_plane[static_cast<size_t>(u)] = vp;
          return vp;
        }
        const int pprod = plane_producer_pw[static_cast<size_t>(vp)];
        if (!bn && pprod >= 0 && p.pw[static_cast<size_t>(pprod)].out2_plane < 0 && p.pw[static_cast<size_t>(pprod)].prog.ln == 0 &&
            !p.pw[static_cast<size_t>(pprod)].concat && !p.pw[static_cast<size_t>(pprod)].dw) {
          PwStep& ps = p.pw[static_cast<size_t>(pprod)];
          int ns = 0, ops[kPwMaxPlanes], affs[kPwMaxPlanes], relus[kPwMaxPlanes];
          if (pw_as_fold(ps.prog, &ns, ops, affs, relus) && ps.prog.n_planes_used == ns) {
            const int np = new_plane(p.planes[static_cast<size_t>(vp)].C, ps.level, true);
            ps.out2_plane = np;
            node_plane[static_cast<size_t>(u)] = np;
            return np;
          }
        }
        const int prod = plane_producer_tc[static_cast<size_t>(vp)];
        if (prod >= 0 && p.tc[static_cast<size_t>(prod)].out_plane == vp && p.tc[static_cast<size_t>(prod)].out2_plane < 0) {
          TcOp& op = p.tc[static_cast<size_t>(prod)];
          const int np = new_plane(p.planes[static_cast<size_t>(vp)].C, op.level, true);
          op.out2_plane = np;
          if (bn) {
            std::vector<float> s, t;
            bn_affine(p.P(bn->gamma), p.P(bn->beta), p.P(bn->rmean), p.P(bn->rvar), s, t);
            s.resize(static_cast<size_t>(op.cout), 0.f);
            t.resize(static_cast<size_t>(op.cout), 0.f);
            op.s2 = p.upload(s);
            op.t2 = p.upload(t);
          }
          plane_producer_tc[static_cast<size_t>(np)] = prod;
          node_plane[static_cast<size_t>(u)] = np;
          return np;
        }
      }
    }
    if (nd.op == CNRX_OP_DWCONV) {
      // depthwise conv (network.hpp:443-449 conv_stage "depthwise"): CUDA cores, fp32 weights, plane in / out
      const int a = plane_for(nd.in0);
      const int C = p.planes[static_cast<size_t>(a)].C;
      const auto& w = p.P(nd.w);
      PwStep st;
      st.dw = true;
      st.plane_ids[0] = a;
      st.n_planes = 1;
      st.prog.C = C;
      st.dw_kh = static_cast<int>(w.dims[0]);
      st.dw_kw = static_cast<int>(w.dims[1]);
      st.dw_dil = nd.dilation_f;
      const int creal = static_cast<int>(w.dims[2]);
      std::vector<float> wp(static_cast<size_t>(st.dw_kh * st.dw_kw * C), 0.f);
      for (int t = 0; t < st.dw_kh * st.dw_kw; ++t)
        for (int c = 0; c < creal; ++c)
          wp[static_cast<size_t>(t * C + c)] = w.data[static_cast<size_t>(t * creal + c)];  // [kh,kw,C,1]
      st.dw_w = p.upload(wp);
      if (nd.b >= 0) {
        std::vector<float> bp(static_cast<size_t>(C), 0.f);
        for (int c = 0; c < creal; ++c) bp[static_cast<size_t>(c)] = p.P(nd.b).data[static_cast<size_t>(c)];
        st.dw_b = p.upload(bp);
      }
      st.level = p.planes[static_cast<size_t>(a)].level + 1;
      st.out_plane = new_plane(C, st.level, false);
      use(a, st.level);
      p.pw.push_back(st);
      plane_producer_pw[static_cast<size_t>(st.out_plane)] = static_cast<int>(p.pw.size()) - 1;
      node_plane[static_cast<size_t>(u)] = st.out_plane;
      return st.out_plane;
    }
    if (nd.op == CNRX_OP_CONCAT) {
      // concat fusion (network.hpp:541-544): the two planes side by side, consumed by the 1x1 restore conv
      const int a = plane_for(nd.in0), b = plane_for(nd.in1);
      const int ca = p.planes[static_cast<size_t>(a)].C, cb = p.planes[static_cast<size_t>(b)].C;
      if (ca != p.N(nd.in0).out_channels || cb != p.N(nd.in1).out_channels || round_cin(ca + cb) != ca + cb)
        throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: concat of " + std::to_string(p.N(nd.in0).out_channels) + " + " +
                                              std::to_string(p.N(nd.in1).out_channels) + " channels");
      PwStep st;
      st.concat = true;
      st.plane_ids[0] = a;
      st.plane_ids[1] = b;
      st.n_planes = 2;
      st.prog.C = ca + cb;
      st.level = std::max(p.planes[static_cast<size_t>(a)].level, p.planes[static_cast<size_t>(b)].level) + 1;
      st.out_plane = new_plane(ca + cb, st.level, false);
      use(a, st.level);
      use(b, st.level);
      p.pw.push_back(st);
      plane_producer_pw[static_cast<size_t>(st.out_plane)] = static_cast<int>(p.pw.size()) - 1;
      node_plane[static_cast<size_t>(u)] = st.out_plane;
      return st.out_plane;
    }
    if (nd.op == CNRX_OP_LN) {
      // layer norm over the channels of each row: the chain feeding it, then the row statistics (generic
      // pointwise kernel, double accumulation like norms.hpp:171-184), output rounded to the plane format
      PwStep st;
      std::vector<std::vector<float>> aff;
      int level = 0;
      if (!build_chain(nd.in0, st, aff, level))
        throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: layer norm input " + std::to_string(nd.in0) +
                                              " is not a linear pointwise chain over planes");
      const int k = static_cast<int>(aff.size()) / 2;
      if (k >= kPwMaxAff) throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: too many affine steps before a layer norm");
      aff.push_back(p.P(nd.gamma).data);
      aff.push_back(p.P(nd.beta).data);
      st.prog.ln = k + 1;
      st.prog.ln_c = nd.out_channels;
      const int C = round_cin(nd.out_channels);
      st.level = level + 1;
      st.out_plane = new_plane(C, st.level, false);
      finish_pw(st, aff, C);
      p.pw.push_back(st);
      plane_producer_pw[static_cast<size_t>(st.out_plane)] = static_cast<int>(p.pw.size()) - 1;
      node_plane[static_cast<size_t>(u)] = st.out_plane;
      return st.out_plane;
    }
    // general linear pointwise chain -> pointwise program kernel
    PwStep st;
    std::vector<std::vector<float>> aff;
    int level = 0;
    if (!build_chain(u, st, aff, level))
      throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: node " + std::to_string(u) + " (" +
                                            std::to_string(nd.op) + ") is not a linear pointwise chain over planes");
    const int C = round_cin(nd.out_channels);
    st.level = level + 1;
    st.out_plane = new_plane(C, st.level, false);
    finish_pw(st, aff, C);
    p.pw.push_back(st);
    plane_producer_pw[static_cast<size_t>(st.out_plane)] = static_cast<int>(p.pw.size()) - 1;
    node_plane[static_cast<size_t>(u)] = st.out_plane;
    return st.out_plane;
  }

  // Pre-activation residual blocks y = conv2(relu(bn(conv1(relu?(x))))) + x over 64-channel planes, when
  // conv1's output feeds nothing but conv2, run as one kernel (conv_blk.cu): same values as the
  // two-kernel path (conv1's output is rounded to 16 bits either way), a third of the HBM bytes.  The
  // default at every batch size (measured faster sustained: less HBM traffic keeps the power-capped
  // clock higher); cnrx_plan_options::fused_blocks = 0 selects the two-kernel program.
  void fuse_blocks() {
    if (p.opt.fused_blocks == 0) return;
    std::vector<int> readers(p.planes.size(), 0);
    for (const auto& op : p.tc) {
      if (op.in_plane >= 0) ++readers[static_cast<size_t>(op.in_plane)];
      if (op.res_plane >= 0) ++readers[static_cast<size_t>(op.res_plane)];
    }
    for (const auto& st : p.pw)
      for (int k = 0; k < st.n_planes; ++k) ++readers[static_cast<size_t>(st.plane_ids[k])];
    for (size_t bi = 0; bi < p.tc.size(); ++bi) {
      TcOp& b = p.tc[bi];
      if (!b.ws || b.relu || b.relu_in || b.res_plane < 0 || b.out2_plane >= 0 || b.stem) continue;
      const int ai = plane_producer_tc[static_cast<size_t>(b.in_plane)];
      if (ai < 0) continue;
      TcOp& a = p.tc[static_cast<size_t>(ai)];
      if (!a.ws || a.fused_away || a.blk_c1 >= 0 || a.out_plane != b.in_plane || !a.relu || a.res_plane >= 0 ||
          a.out2_plane >= 0 || a.dil != b.dil || a.in_plane != b.res_plane || a.stem)
        continue;
      if (readers[static_cast<size_t>(a.out_plane)] != 1) continue;
      b.blk_c1 = ai;
      a.fused_away = true;
    }
  }

  // The CoNet interaction + LLR head folded into the epilogue of the subnetworks' last convs
  // (conv_ws.cu kWsHead) when the head is a fold over 64-channel planes each written by a 64->64
  // weights-stationary conv (residual epilogue, no other reader), all in one launch group.  The
  // two-kernel program then skips the head kernel; the fused-block program (small batches) keeps it.
  // Both compute z the same way and run the same head UMMAs, so their LLRs are identical.
  // Opt-in while it is slower than conv + head kernel (cnrx_plan_options::fused_head; bf16 plans only:
  // the fused epilogue runs the head on the tensor core over 16-bit z).
  void fuse_head() {
    if (p.opt.fused_head != 1 || p.fp16 || p.opt.tensor_core_head == 0) return;
    const int hk = static_cast<int>(p.pw.size()) - 1;
    if (hk < 0) return;
    const PwStep& hs = p.pw[static_cast<size_t>(hk)];
    int ns = 0, ops[kPwMaxPlanes], affs[kPwMaxPlanes], relus[kPwMaxPlanes];
    if (hs.out_plane >= 0 || hs.prog.C != 64 || hs.prog.head_bits > 8 || hs.prog.head_bits < 1) return;
    const int nb = hs.prog.head_bits;
    if (nb != 2 && nb != 4 && nb != 6 && nb != 8) return;  // head.cu's variants (identical results)
    if (!pw_as_fold(hs.prog, &ns, ops, affs, relus) || hs.prog.n_planes_used != ns || ns < 1 || ns > 3) return;
    std::vector<int> readers(p.planes.size(), 0);
    for (const auto& op : p.tc) {
      if (op.in_plane >= 0) ++readers[static_cast<size_t>(op.in_plane)];
      if (op.res_plane >= 0) ++readers[static_cast<size_t>(op.res_plane)];
    }
    for (const auto& st : p.pw)
      for (int k = 0; k < st.n_planes; ++k) ++readers[static_cast<size_t>(st.plane_ids[k])];
    std::vector<int> prod(static_cast<size_t>(ns));
    for (int k = 0; k < ns; ++k) {
      const int pl = hs.plane_ids[k];
      const int t = plane_producer_tc[static_cast<size_t>(pl)];
      if (t < 0 || readers[static_cast<size_t>(pl)] != 1) return;
      const TcOp& op = p.tc[static_cast<size_t>(t)];
      if (!op.ws || op.stem || op.fused_away || op.out_plane != pl || op.out2_plane >= 0 || op.relu || op.relu_in ||
          op.res_plane < 0)
        return;
      prod[static_cast<size_t>(k)] = t;
    }
    const int lv = p.tc[static_cast<size_t>(prod[0])].level;
    auto& groups = p.tc_groups_by_level[static_cast<size_t>(lv)];
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      auto& grp = groups[gi];
      if (static_cast<int>(grp.size()) != ns) continue;
      bool all = true;
      for (int t : prod)
        if (std::find(grp.begin(), grp.end(), t) == grp.end()) all = false;
      if (!all) continue;
      grp = prod;  // launch member r = fold operand r (cluster rank r)
      p.hf_level = lv;
      p.hf_group = static_cast<int>(gi);
      p.hf_pw = hk;
      WsHead& h = p.hf;
      std::memset(&h, 0, sizeof(h));
      h.ns = ns;
      h.nb = nb;
      for (int k = 0; k < ns; ++k) {
        h.op[k] = ops[k];
        h.relu[k] = relus[k];
        h.aff_s[k] = affs[k] >= 0 ? hs.prog.aff_s[affs[k]] : nullptr;
        h.aff_t[k] = affs[k] >= 0 ? hs.prog.aff_t[affs[k]] : nullptr;
      }
      h.w = hs.prog.head_w;
      h.b = hs.prog.head_b;
      return;
    }
  }

  // The CoNet interaction + LLR head folded into the subnetworks' last fused residual blocks (conv_blk.cu
  // BlkFold, fused-block program): the head is a fold over 64-channel planes each written by the conv2 of
  // a fused block (ReLU'd block input, residual, no other reader) of one launch group.  The group then
  // runs as one launch per subnetwork in fold order (ensure_workspace builds the chain); LLRs equal the
  // separate head kernel's fp32 GEMV path bit for bit.  cnrx_plan_options::fused_head.
  void fuse_head_blk() {
    if (p.opt.fused_head != 1 || p.opt.fused_blocks == 0) return;
    const int hk = static_cast<int>(p.pw.size()) - 1;
    if (hk < 0) return;
    const PwStep& hs = p.pw[static_cast<size_t>(hk)];
    int ns = 0, ops[kPwMaxPlanes], affs[kPwMaxPlanes], relus[kPwMaxPlanes];
    if (hs.out_plane >= 0 || hs.prog.C != 64 || hs.prog.head_bits < 1 || hs.prog.head_bits > 8) return;
    if (!pw_as_fold(hs.prog, &ns, ops, affs, relus) || hs.prog.n_planes_used != ns || ns < 2 || ns > 4) return;
    std::vector<int> readers(p.planes.size(), 0);
    for (const auto& op : p.tc) {
      if (op.in_plane >= 0) ++readers[static_cast<size_t>(op.in_plane)];
      if (op.res_plane >= 0) ++readers[static_cast<size_t>(op.res_plane)];
    }
    for (const auto& st : p.pw)
      for (int k = 0; k < st.n_planes; ++k) ++readers[static_cast<size_t>(st.plane_ids[k])];
    std::vector<int> prod(static_cast<size_t>(ns));
    for (int k = 0; k < ns; ++k) {
      const int pl = hs.plane_ids[k];
      const int t = plane_producer_tc[static_cast<size_t>(pl)];
      if (t < 0 || readers[static_cast<size_t>(pl)] != 1) return;
      const TcOp& op = p.tc[static_cast<size_t>(t)];
      if (op.blk_c1 < 0 || op.out_plane != pl || op.out2_plane >= 0 || op.relu || op.res_plane < 0) return;
      if (!p.tc[static_cast<size_t>(op.blk_c1)].relu_in) return;  // fold epilogues exist for ReLU'd inputs
      prod[static_cast<size_t>(k)] = t;
    }
    const int lv = p.tc[static_cast<size_t>(prod[0])].level;
    auto& groups = p.tc_groups_by_level[static_cast<size_t>(lv)];
    for (size_t gi = 0; gi < groups.size(); ++gi) {
      auto& grp = groups[gi];
      if (static_cast<int>(grp.size()) != ns) continue;
      bool all = true;
      for (int t : prod)
        if (std::find(grp.begin(), grp.end(), t) == grp.end()) all = false;
      if (!all) continue;
      p.hb_level = lv;
      p.hb_group = static_cast<int>(gi);
      p.hb_pw = hk;
      p.hb_ns = ns;
      for (int k = 0; k < ns; ++k) {
        p.hb_ops[k] = ops[k];
        p.hb_affs[k] = affs[k];
        p.hb_relus[k] = relus[k];
        p.hb_tc[k] = prod[static_cast<size_t>(k)];
      }
      return;
    }
  }

  void compile() {
    const int n = static_cast<int>(p.nodes.size());
    node_plane.assign(static_cast<size_t>(n), -1);
    std::vector<char> absorbed(static_cast<size_t>(n), 0);
    const int cin0 = round_cin(p.in_ch);
    node_plane[static_cast<size_t>(p.in_node)] = new_plane(cin0, 0, false);
    for (int i = 0; i < n; ++i) {
      const cnrx_node& nd = p.N(i);
      if (nd.op != CNRX_OP_CONV || absorbed[static_cast<size_t>(i)] || i == p.out_node) continue;
      const auto& w = p.P(nd.w);
      TcOp op;
      op.node = i;
      op.ks = static_cast<int>(w.dims[0]);
      require(w.dims[0] == w.dims[1], "bf16 plan supports square kernels only");
      if (op.ks != 1 && op.ks != 3)
        throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan supports 1x1 and 3x3 convolutions");
      op.dil = nd.dilation_f;
      // relu(v) feeding a 64->64 3x3 conv (weights-stationary kernel) or a 96->96 one (CTA-pair kernel):
      // the conv applies the ReLU to its input window in shared memory, so v's producer need not store a
      // second, pre-activated plane (relu commutes with the 16-bit rounding: identical values).
      const bool no_relu_in = p.opt.relu_on_load == 0;
      {
        const cnrx_node& in = p.N(nd.in0);
        const int v = in.op == CNRX_OP_RELU ? in.in0 : -1;
        const int vC = v >= 0 && node_plane[static_cast<size_t>(v)] >= 0
                           ? p.planes[static_cast<size_t>(node_plane[static_cast<size_t>(v)])].C : 0;
        const bool ws64 = w.dims[2] == 64 && w.dims[3] == 64 && vC == 64 && p.opt.weights_stationary;
        const bool pair96 = round_cin(static_cast<int>(w.dims[2])) == 96 && round_cout(static_cast<int>(w.dims[3])) == 96 &&
                            vC == 96 && p.opt.cta_pair;
        // split plans: every 3x3 conv (conv_x3.cu has a ReLU warp for its (hi, lo) windows)
        const bool x3 = p.split && vC > 0;
        if (!no_relu_in && v >= 0 && node_plane[static_cast<size_t>(nd.in0)] < 0 && node_plane[static_cast<size_t>(v)] >= 0 &&
            !p.planes[static_cast<size_t>(node_plane[static_cast<size_t>(v)])].nonneg && op.ks == 3 && (ws64 || pair96 || x3)) {
          op.relu_in = 1;
          op.in_plane = node_plane[static_cast<size_t>(v)];
        } else {
          op.in_plane = plane_for(nd.in0);
        }
      }
      op.cin = p.planes[static_cast<size_t>(op.in_plane)].C;
      op.cout = round_cout(nd.out_channels);
      op.cin_real = static_cast<int>(w.dims[2]);
      op.cout_real = static_cast<int>(w.dims[3]);
      if (!(p.split ? conv_x3_supported(op.cin, op.cout, op.ks) : conv_tc_supported(op.cin, op.cout, op.ks)))
        throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: no tcgen05 conv for cin=" + std::to_string(op.cin) +
                                              " cout=" + std::to_string(op.cout) + " k=" + std::to_string(op.ks));
      // epilogue absorption: [BN] [ReLU] [add residual]
      std::vector<float> scale, shift;
      std::vector<float> bias(static_cast<size_t>(op.cout), 0.f);
      if (nd.b >= 0)
        for (int c = 0; c < nd.out_channels; ++c) bias[static_cast<size_t>(c)] = p.P(nd.b).data[static_cast<size_t>(c)];
      int end = i;
      int c = p.single_consumer(end);
      if (c >= 0 && p.N(c).op == CNRX_OP_BN && c != p.out_node) {
        const auto& bn = p.N(c);
        bn_affine(p.P(bn.gamma), p.P(bn.beta), p.P(bn.rmean), p.P(bn.rvar), scale, shift);
        for (int k = 0; k < nd.out_channels; ++k)
          bias[static_cast<size_t>(k)] = bias[static_cast<size_t>(k)] * scale[static_cast<size_t>(k)] + shift[static_cast<size_t>(k)];
        absorbed[static_cast<size_t>(c)] = 1;
        end = c;
        c = p.single_consumer(end);
      }
      if (c >= 0 && p.N(c).op == CNRX_OP_RELU) {
        op.relu = 1;
        absorbed[static_cast<size_t>(c)] = 1;
        end = c;
        c = p.single_consumer(end);
      }
      if (!op.relu && c >= 0 && p.N(c).op == CNRX_OP_ADD) {
        const int other = p.N(c).in0 == end ? p.N(c).in1 : p.N(c).in0;
        if (other != end && other < i) {
          op.res_plane = plane_for(other);
          if (p.planes[static_cast<size_t>(op.res_plane)].C == op.cout) {
            absorbed[static_cast<size_t>(c)] = 1;
            end = c;
          } else {
            op.res_plane = -1;
          }
        }
      }
      int level = p.planes[static_cast<size_t>(op.in_plane)].level;
      if (op.res_plane >= 0) level = std::max(level, p.planes[static_cast<size_t>(op.res_plane)].level);
      op.level = level + 1;
      use(op.in_plane, op.level);
      if (op.res_plane >= 0) use(op.res_plane, op.level);
      // weights (BN scale folded per output channel) and bias
      op.ws = p.opt.weights_stationary != 0 && op.ks == 3 && op.cin_real == 64 && op.cout_real == 64 && op.cin == 64 && op.cout == 64;
      if (op.relu_in && !op.ws && !p.split && !(op.cin == 96 && op.cout == 96 && op.ks == 3))
        throw Error(CNRX_ERR_UNSUPPORTED, "internal: relu-on-load needs the ws or the CTA-pair conv kernel");
      if (op.ws) {
        std::vector<uint32_t> img(conv_ws64_wimg_bytes() / 4);
        conv_ws64_pack_weights(w.data.data(), scale.empty() ? nullptr : scale.data(), p.fp16, img.data());
        op.wimg = p.upload_bytes(img.data(), img.size() * 4);
      } else if (p.split) {
        std::vector<uint8_t> img(conv_x3_wimg_bytes(op.cin, op.cout, op.ks));
        conv_x3_pack_weights(w.data.data(), op.ks, static_cast<int>(w.dims[2]), static_cast<int>(w.dims[3]),
                             scale.empty() ? nullptr : scale.data(), op.cin, op.cout, p.fp16, img.data());
        op.wimg = p.upload_bytes(img.data(), img.size());
      } else {
        std::vector<uint8_t> img(conv_tc_wimg_bytes(op.cin, op.cout, op.ks));
        conv_tc_pack_weights(w.data.data(), op.ks, static_cast<int>(w.dims[2]), static_cast<int>(w.dims[3]),
                             scale.empty() ? nullptr : scale.data(), op.cin, op.cout, p.fp16, img.data());
        op.wimg = p.upload_bytes(img.data(), img.size());
      }
      op.bias = p.upload(bias);
      if (op.in_plane == 0 && op.ks == 1 && op.res_plane < 0 && stem_supported_cin(op.cin_real) &&
          op.cout_real % 8 == 0 && op.cout_real <= 64 && op.cout == op.cout_real) {
        std::vector<float> wf(static_cast<size_t>(op.cin_real) * op.cout_real);
        for (int ci = 0; ci < op.cin_real; ++ci)
          for (int co = 0; co < op.cout_real; ++co)
            wf[static_cast<size_t>(ci) * op.cout_real + co] =
                w.data[static_cast<size_t>(ci) * op.cout_real + co] * (scale.empty() ? 1.f : scale[static_cast<size_t>(co)]);
        op.stem_w = p.upload(wf);
      }
      op.out_plane = new_plane(op.cout, op.level, op.relu != 0);
      p.tc.push_back(op);
      plane_producer_tc[static_cast<size_t>(op.out_plane)] = static_cast<int>(p.tc.size()) - 1;
      node_plane[static_cast<size_t>(end)] = op.out_plane;
    }
    // output: 1x1 conv head over a linear pointwise chain (pointwise program / TMA head kernel), or a 3x3
    // head (NetSpec.kernel = 3, network.hpp:559) as a tensor-core conv over the chain's plane whose epilogue
    // writes the fp32 LLRs
    const cnrx_node& on = p.N(p.out_node);
    if (on.op != CNRX_OP_CONV) throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: output node must be a conv");
    const auto& hw = p.P(on.w);
    if (hw.dims[0] == 3 && hw.dims[1] == 3 && on.out_channels <= 32) {
      TcOp op;
      op.node = p.out_node;
      op.ks = 3;
      op.dil = on.dilation_f;
      op.llr_head = true;
      op.in_plane = plane_for(on.in0);
      op.cin = p.planes[static_cast<size_t>(op.in_plane)].C;
      op.cout = round_cout(on.out_channels);
      op.cin_real = static_cast<int>(hw.dims[2]);
      op.cout_real = static_cast<int>(hw.dims[3]);
      if (!(p.split ? conv_x3_supported(op.cin, op.cout, 3) : conv_tc_supported(op.cin, op.cout, 3)))
        throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: no tcgen05 conv for the 3x3 head (cin=" + std::to_string(op.cin) + ")");
      if (p.split) {
        std::vector<uint8_t> img(conv_x3_wimg_bytes(op.cin, op.cout, 3));
        conv_x3_pack_weights(hw.data.data(), 3, op.cin_real, op.cout_real, nullptr, op.cin, op.cout, p.fp16, img.data());
        op.wimg = p.upload_bytes(img.data(), img.size());
      } else {
        std::vector<uint8_t> img(conv_tc_wimg_bytes(op.cin, op.cout, 3));
        conv_tc_pack_weights(hw.data.data(), 3, op.cin_real, op.cout_real, nullptr, op.cin, op.cout, p.fp16, img.data());
        op.wimg = p.upload_bytes(img.data(), img.size());
      }
      std::vector<float> hbias(static_cast<size_t>(op.cout), 0.f);
      if (on.b >= 0)
        for (int c = 0; c < on.out_channels; ++c) hbias[static_cast<size_t>(c)] = p.P(on.b).data[static_cast<size_t>(c)];
      op.bias = p.upload(hbias);
      op.level = p.planes[static_cast<size_t>(op.in_plane)].level + 1;
      use(op.in_plane, op.level);
      p.tc.push_back(op);
      finish_schedule();
      return;
    }
    if (hw.dims[0] != 1 || hw.dims[1] != 1 || on.out_channels > kPwMaxBits)
      throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: output conv must be 1x1 (or 3x3) with <= 16 outputs");
    PwStep st;
    std::vector<std::vector<float>> aff;
    int level = 0;
    if (!build_chain(on.in0, st, aff, level))
      throw Error(CNRX_ERR_UNSUPPORTED, "bf16 plan: head input is not a linear pointwise chain over planes");
    st.level = level + 1;
    st.out_plane = -1;
    const int C = round_cin(static_cast<int>(hw.dims[2]));
    for (int k = 0; k < st.n_planes; ++k)
      require(p.planes[static_cast<size_t>(st.plane_ids[k])].C == C, "bf16 plan: head operand channel mismatch");
    std::vector<float> wpad(static_cast<size_t>(C) * on.out_channels, 0.f);
    for (int ci = 0; ci < hw.dims[2]; ++ci)
      for (int co = 0; co < on.out_channels; ++co)
        wpad[static_cast<size_t>(ci) * on.out_channels + co] = hw.data[static_cast<size_t>(ci) * on.out_channels + co];
    std::vector<float> hb(static_cast<size_t>(on.out_channels), 0.f);
    if (on.b >= 0) hb = p.P(on.b).data;
    st.prog.head_bits = on.out_channels;
    st.prog.tc_head = !p.fp16 && p.opt.tensor_core_head != 0;
    st.prog.head_w = p.upload(wpad);
    st.prog.head_b = p.upload(hb);
    finish_pw(st, aff, C);
    p.pw.push_back(st);
    finish_schedule();
  }

  // residual-block fusion, level schedule, launch groups, fused heads, buffer assignment
  void finish_schedule() {
    fuse_blocks();
    // level schedule
    int maxl = 0;
    for (auto& op : p.tc) maxl = std::max(maxl, op.level);
    for (auto& s2 : p.pw) maxl = std::max(maxl, s2.level);
    p.n_levels = maxl + 1;
    p.tc_groups_by_level.assign(static_cast<size_t>(p.n_levels), {});
    p.pw_by_level.assign(static_cast<size_t>(p.n_levels), {});
    // The CUDA-core fused featurize+stem kernel is opt-in (cuda_core_stem): measured slower than
    // featurize + the tensor-core 1x1 conv at cfg2 sizes (profiles/r01_session2_notes.md).
    const bool no_stem = p.opt.cuda_core_stem == 0;
    for (int k = 0; k < static_cast<int>(p.tc.size()); ++k) {
      TcOp& op = p.tc[static_cast<size_t>(k)];
      if (!no_stem && op.stem_w && static_cast<int>(p.stem_ops.size()) < kStemMaxOps &&
          (p.stem_ops.empty() || p.tc[static_cast<size_t>(p.stem_ops[0])].cin_real == op.cin_real)) {
        op.stem = true;
        p.stem_ops.push_back(k);
      }
    }
    p.need_plane0 = false;
    for (const auto& op : p.tc)
      if (!op.stem && (op.in_plane == 0 || op.res_plane == 0)) p.need_plane0 = true;
    for (const auto& st2 : p.pw)
      for (int k = 0; k < st2.n_planes; ++k)
        if (st2.plane_ids[k] == 0) p.need_plane0 = true;
    for (int k = 0; k < static_cast<int>(p.tc.size()); ++k) {
      const TcOp& op = p.tc[static_cast<size_t>(k)];
      if (op.stem) continue;
      auto& groups = p.tc_groups_by_level[static_cast<size_t>(op.level)];
      bool placed = false;
      for (auto& g : groups) {
        const TcOp& o0 = p.tc[static_cast<size_t>(g[0])];
        const bool blk0 = o0.blk_c1 >= 0, blk = op.blk_c1 >= 0;
        if (static_cast<int>(g.size()) < kTcMaxGroups && o0.cin == op.cin && o0.cout == op.cout && o0.ks == op.ks &&
            !o0.llr_head && !op.llr_head &&
            o0.ws == op.ws && blk0 == blk && o0.fused_away == op.fused_away && (op.ws || o0.relu_in == op.relu_in) &&
            (!blk || p.tc[static_cast<size_t>(o0.blk_c1)].relu_in == p.tc[static_cast<size_t>(op.blk_c1)].relu_in)) {
          g.push_back(k);
          placed = true;
          break;
        }
      }
      if (!placed) groups.push_back({k});
    }
    for (int k = 0; k < static_cast<int>(p.pw.size()); ++k)
      p.pw_by_level[static_cast<size_t>(p.pw[static_cast<size_t>(k)].level)].push_back(k);
    fuse_head();
    fuse_head_blk();
    // out2 planes share their producer's level; every plane is live from its level to last use
    for (auto& op : p.tc) {
      if (op.out2_plane >= 0) p.planes[static_cast<size_t>(op.out2_plane)].level = op.level;
    }
    for (auto& st2 : p.pw) {
      if (st2.out2_plane >= 0) p.planes[static_cast<size_t>(st2.out2_plane)].level = st2.level;
    }
    // buffer assignment by liveness over levels (a buffer is reusable once every reader's level passed)
    std::vector<int> order(p.planes.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = static_cast<int>(k);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return p.planes[static_cast<size_t>(a)].level < p.planes[static_cast<size_t>(b)].level;
    });
    std::vector<int> buf_free_after;
    for (int pl : order) {
      auto& pi = p.planes[static_cast<size_t>(pl)];
      if (pi.last_use < pi.level) pi.last_use = pi.level;
      int chosen = -1;
      for (size_t b = 0; b < p.buf_channels.size(); ++b)
        if (p.buf_channels[b] == pi.C && buf_free_after[b] < pi.level) {
          chosen = static_cast<int>(b);
          break;
        }
      if (chosen < 0) {
        chosen = static_cast<int>(p.buf_channels.size());
        p.buf_channels.push_back(pi.C);
        buf_free_after.push_back(-1);
      }
      pi.buffer = chosen;
      buf_free_after[static_cast<size_t>(chosen)] = pi.last_use;
    }
  }
};

// ------------------------------------------------------------------------------------------------
// Execution
// ------------------------------------------------------------------------------------------------
void ensure_workspace_impl(cnrx_plan& p, int B, int T, int F);

// A failed (re)build (batch too large for one plane, out of device memory) leaves no half-built
// workspace behind: the next call rebuilds from scratch.
void ensure_workspace(cnrx_plan& p, int B, int T, int F) {
  Workspace& ws = p.ws;
  if (ws.B == B && ws.T == T && ws.F == F) return;
  if (p.precision != CNRX_FP32) make_geom(B, T, F, p.npad);  // validate before touching any state
  try {
    ensure_workspace_impl(p, B, T, F);
  } catch (...) {
    for (void* b : ws.buffers) ws_free(ws, b);
    ws.buffers.clear();
    ws.sizes.clear();
    ws.launches.clear();
    ws.cap_B = 0;
    ws.B = ws.T = ws.F = -1;
    throw;
  }
}

void ensure_workspace_impl(cnrx_plan& p, int B, int T, int F) {
  Workspace& ws = p.ws;
  // A smaller batch of the same grid reuses the buffers (capacity cap_B): only the geometry and the
  // launch descriptors change.  Every producer writes all rows of [0, Nalloc) (zeros on padding rows)
  // and TMA zero-fills past the descriptor's Nalloc, so stale rows beyond it are never read.
  const bool reuse = ws.T == T && ws.F == F && B <= ws.cap_B;
  ws.launches.clear();
  if (p.gexec) {
    cudaGraphExecDestroy(p.gexec);
    p.gexec = nullptr;
    p.gkey.clear();
  }
  if (!reuse) {
    for (void* b : ws.buffers) ws_free(ws, b);
    ws.buffers.clear();
    ws.sizes.clear();
    ws.cap_B = B;
  }
  ws.B = B;
  ws.T = T;
  ws.F = F;
  if (p.precision == CNRX_FP32) {
    if (reuse) return;
    const int64_t rows = static_cast<int64_t>(B) * T * F;
    for (int c : p.f32_buf_channels) {
      ws.buffers.push_back(ws_malloc(ws, static_cast<size_t>(rows) * c * sizeof(float)));
    }
    return;
  }
  ws.geo = make_geom(B, T, F, p.npad);
  if (!reuse)
    for (int c : p.buf_channels) {
      const size_t bytes = static_cast<size_t>(ws.geo.Nalloc) * c * 2 * (p.split ? 2 : 1);
      ws.buffers.push_back(ws_malloc(ws, bytes));  // every producer writes all rows of [0, Nalloc): no clearing needed
    }
  // tensor maps / launch descriptors per TC group
  auto plane_ptr = [&](int pl) -> __nv_bfloat16* {
    return pl < 0 ? nullptr
                  : static_cast<__nv_bfloat16*>(ws.buffers[static_cast<size_t>(p.planes[static_cast<size_t>(pl)].buffer)]);
  };
  // fused residual blocks (every batch size by default), if every block's window fits
  bool fused = p.opt.fused_blocks != 0;
  {
    for (const auto& op : p.tc)
      if (op.blk_c1 >= 0 && !conv_blk64_supported_halo(ws.geo.T1 * op.dil + 1)) fused = false;
  }
  ws.blocks_fused = fused;
  ws.head_fused = false;
  ws.head_blk_fused = false;
  for (int lv = 0; lv < p.n_levels; ++lv)
    for (size_t gidx = 0; gidx < p.tc_groups_by_level[static_cast<size_t>(lv)].size(); ++gidx) {
      auto& grp = p.tc_groups_by_level[static_cast<size_t>(lv)][gidx];
      Workspace::GroupLaunch GL;
      const TcOp& op0 = p.tc[static_cast<size_t>(grp[0])];
      GL.ws = op0.ws;
      GL.skip = fused && op0.fused_away;
      GL.blk = fused && op0.blk_c1 >= 0;
      if (GL.skip) {
        ws.launches.push_back(GL);
        continue;
      }
      if (GL.blk) {
        BlkLaunch& L = GL.blkl;
        std::memset(&L, 0, sizeof(L));
        L.geo = ws.geo;
        L.ngroups = static_cast<int>(grp.size());
        L.n_tiles = conv_blk64_tiles(ws.geo.Nalloc);
        L.relu_in = p.tc[static_cast<size_t>(op0.blk_c1)].relu_in;
        L.fp16 = p.fp16;
        // a non-negative input (the stem's ReLU output) also runs the ReLU-copy variant (identity ReLU,
        // same values): measured ~0.5 % faster for cfg2's first block
        {
          bool nonneg = true;
          for (int k : grp) nonneg = nonneg && p.planes[static_cast<size_t>(p.tc[static_cast<size_t>(p.tc[static_cast<size_t>(k)].blk_c1)].in_plane)].nonneg;
          if (!L.relu_in && nonneg) L.relu_in = 1;
        }
        int win_alloc = 0;
        for (size_t gi = 0; gi < grp.size(); ++gi) {
          const TcOp& c2 = p.tc[static_cast<size_t>(grp[gi])];
          const TcOp& c1 = p.tc[static_cast<size_t>(c2.blk_c1)];
          BlkGroup& g = L.g[gi];
          g.dil = c1.dil;
          g.halo = ws.geo.T1 * c1.dil + 1;
          win_alloc = std::max(win_alloc, conv_blk64_win_alloc(g.halo));
          conv_blk64_make_maps(plane_ptr(c1.in_plane), plane_ptr(c2.out_plane), ws.geo.Nalloc, &g);
          g.wimg1 = static_cast<const uint32_t*>(c1.wimg);
          g.wimg2 = static_cast<const uint32_t*>(c2.wimg);
          g.bias1 = c1.bias;
          g.bias2 = c2.bias;
        }
        L.win_alloc = win_alloc;
        L.xstages = conv_blk64_xstages(win_alloc, L.relu_in);
        if (L.xstages == 0) throw Error(CNRX_ERR_UNSUPPORTED, "fused residual block exceeds shared memory (fused_blocks = 0)");
        if (lv == p.hb_level && static_cast<int>(gidx) == p.hb_group) {
          // interaction + head folded into these blocks: one launch per subnetwork, in fold order
          const PwProgram& hp = p.pw[static_cast<size_t>(p.hb_pw)].prog;
          const size_t fbytes = conv_blk64_part_bytes(ws.geo.Nalloc);
          const int nbuf = p.hb_ns > 3 ? 2 : (p.hb_ns > 2 ? 1 : 0);
          if (ws.fold_bytes < fbytes) {
            for (void*& b : ws.fold_bufs) {
              ws_free(ws, b);
              b = nullptr;
            }
            ws.fold_bytes = 0;
            for (int i = 0; i < nbuf; ++i) ws.fold_bufs[i] = ws_malloc(ws, fbytes);
            ws.fold_bytes = fbytes;
          }
          for (int k = 0; k < p.hb_ns; ++k) {
            size_t gi = 0;
            while (grp[gi] != p.hb_tc[k]) ++gi;
            BlkLaunch C = L;
            C.ngroups = 1;
            C.g[0] = L.g[gi];
            C.epi = k == 0 ? 0 : (k == p.hb_ns - 1 ? 2 : 1);
            if (C.epi) {
              BlkFold& f = C.fold;
              std::memset(&f, 0, sizeof(f));
              const bool f32 = k >= 2;
              // mid launch k writes partial buffer (k - 1) & 1; launch k >= 2 reads (k - 2) & 1
              const void* opnd = f32 ? ws.fold_bufs[(k - 2) & 1]
                                     : plane_ptr(p.tc[static_cast<size_t>(p.hb_tc[0])].out_plane);
              void* pout = C.epi == 1 ? ws.fold_bufs[(k - 1) & 1] : nullptr;
              if (!opnd || (C.epi == 1 && !pout)) throw Error(CNRX_ERR_CUDA, "internal: fused-block head buffers");
              conv_blk64_make_fold_maps(opnd, f32, pout, ws.geo.Nalloc, &f);
              f.s_prev = p.hb_affs[0] >= 0 ? hp.aff_s[p.hb_affs[0]] : nullptr;
              f.t_prev = p.hb_affs[0] >= 0 ? hp.aff_t[p.hb_affs[0]] : nullptr;
              f.relu_prev = p.hb_relus[0];
              f.op = p.hb_ops[k];
              f.s = p.hb_affs[k] >= 0 ? hp.aff_s[p.hb_affs[k]] : nullptr;
              f.t = p.hb_affs[k] >= 0 ? hp.aff_t[p.hb_affs[k]] : nullptr;
              f.relu = p.hb_relus[k];
              f.head_w = hp.head_w;
              f.head_b = hp.head_b;
              f.nb = hp.head_bits;
              f.dbg = std::getenv("CNRX_FOLD_DEBUG") ? std::atoi(std::getenv("CNRX_FOLD_DEBUG")) : 0;
              C.xstages = conv_blk64_xstages(win_alloc, C.relu_in, C.epi);
              if (C.xstages == 0) throw Error(CNRX_ERR_UNSUPPORTED, "fused-block head exceeds shared memory");
            }
            GL.chain.push_back(C);
          }
          ws.head_blk_fused = true;
        }
      } else if (op0.ws) {
        WsLaunch& L = GL.wsl;
        std::memset(&L, 0, sizeof(L));
        L.fp16 = p.fp16;
        L.geo = ws.geo;
        L.ngroups = static_cast<int>(grp.size());
        L.n_tiles = conv_ws64_tiles(ws.geo.Nalloc);
        int win_alloc = 0;
        for (size_t gi = 0; gi < grp.size(); ++gi) {
          const TcOp& op = p.tc[static_cast<size_t>(grp[gi])];
          WsGroup& g = L.g[gi];
          g.halo = ws.geo.T1 * op.dil + 1;
          g.dil = op.dil;
          win_alloc = std::max(win_alloc, conv_ws64_win_alloc(g.halo));
          conv_ws64_make_maps(plane_ptr(op.in_plane), plane_ptr(op.res_plane), plane_ptr(op.out_plane),
                              plane_ptr(op.out2_plane), ws.geo.Nalloc, &g);
          g.wimg = static_cast<const uint32_t*>(op.wimg);
          g.bias = op.bias;
          g.s2 = op.s2;
          g.t2 = op.t2;
          g.relu = op.relu;
          g.relu_in = op.relu_in;
        }
        L.win_alloc = win_alloc;
        const bool head = !fused && lv == p.hf_level && static_cast<int>(gidx) == p.hf_group;
        int stages = 4;
        while (stages > 1 && (head ? conv_ws64_head_smem_bytes(stages, win_alloc) : conv_ws64_smem_bytes(stages, win_alloc)) >
                                 227 * 1024)
          --stages;
        L.stages = stages;
        if (head) {
          L.head_on = 1;
          L.head = p.hf;
          ws.head_fused = true;
        }
      } else if (p.split) {
        GL.x3 = true;
        X3Launch& L = GL.x3l;
        std::memset(&L, 0, sizeof(L));
        L.fp16 = p.fp16;
        L.geo = ws.geo;
        L.ngroups = static_cast<int>(grp.size());
        if (L.ngroups > kX3MaxGroups) throw Error(CNRX_ERR_UNSUPPORTED, "internal: split conv group too large");
        int win_alloc = 0;
        for (size_t gi = 0; gi < grp.size(); ++gi) {
          const TcOp& op = p.tc[static_cast<size_t>(grp[gi])];
          X3Group& g = L.g[gi];
          g.halo = op.ks == 1 ? 0 : ws.geo.T1 * op.dil + 1;
          g.dil = op.dil;
          win_alloc = std::max(win_alloc, (128 + 2 * g.halo + 31) / 32 * 32);
          conv_x3_make_maps(plane_ptr(op.in_plane), ws.geo.Nalloc, op.cin, g.map);
          g.wimg = static_cast<const uint8_t*>(op.wimg);
          g.bias = op.bias;
          g.res = plane_ptr(op.res_plane);
          g.out = plane_ptr(op.out_plane);
          g.out2 = plane_ptr(op.out2_plane);
          g.s2 = op.s2;
          g.t2 = op.t2;
          g.relu = op.relu;
          g.nb = op.llr_head ? op.cout_real : 0;  // (the LLR pointer is the forward's output, set per call)
          if (op.relu_in) L.relu_in = 1;  // a launch group shares relu_in (grouping rule)
        }
        L.win_alloc = win_alloc;
        if (!conv_x3_config(op0.cin, op0.cout, op0.ks, win_alloc, &L.stages, &L.nslots))
          throw Error(CNRX_ERR_UNSUPPORTED, "split-precision conv working set exceeds shared memory");
      } else {
        TcLaunch& L = GL.tc;
        std::memset(&L, 0, sizeof(L));
        L.fp16 = p.fp16;
        L.geo = ws.geo;
        L.ngroups = static_cast<int>(grp.size());
        int win_alloc = 0;
        for (size_t gi = 0; gi < grp.size(); ++gi) {
          const TcOp& op = p.tc[static_cast<size_t>(grp[gi])];
          TcGroup& g = L.g[gi];
          g.halo = op.ks == 1 ? 0 : ws.geo.T1 * op.dil + 1;
          g.dil = op.dil;
          const int rows = 128 + 2 * g.halo;
          win_alloc = std::max(win_alloc, (rows + 31) / 32 * 32);
          conv_tc_make_maps(plane_ptr(op.in_plane), ws.geo.Nalloc, op.cin, 32, g.map);
          if (conv_tc_staged(op.cin, op.cout)) {
            conv_tc_make_row_map(plane_ptr(op.res_plane), ws.geo.Nalloc, op.cout, &g.res_map);
            conv_tc_make_row_map(plane_ptr(op.out_plane), ws.geo.Nalloc, op.cout, &g.out_map);
            conv_tc_make_row_map(plane_ptr(op.out2_plane), ws.geo.Nalloc, op.cout, &g.out2_map);
          }
          g.wimg = static_cast<const uint8_t*>(op.wimg);
          g.bias = op.bias;
          g.res = plane_ptr(op.res_plane);
          g.out = plane_ptr(op.out_plane);
          g.out2 = plane_ptr(op.out2_plane);
          g.s2 = op.s2;
          g.t2 = op.t2;
          g.relu = op.relu;
          g.nb = op.llr_head ? op.cout_real : 0;  // (the LLR pointer is the forward's output, set per call)
        }
        L.win_alloc = win_alloc;
        bool relu_in = false;
        for (size_t gi = 0; gi < grp.size(); ++gi) {
          const TcOp& op = p.tc[static_cast<size_t>(grp[gi])];
          if (op.res_plane >= 0) L.flags |= 1;
          if (op.out2_plane >= 0) L.flags |= 2;
          relu_in = relu_in || op.relu_in;
        }
        // 96 -> 96 3x3 convs run on CTA pairs (cta_pair = 0: the single-CTA kernel)
        const bool no_pair = p.opt.cta_pair == 0;
        int max_halo = 0;
        for (int k : grp) max_halo = std::max(max_halo, ws.geo.T1 * p.tc[static_cast<size_t>(k)].dil + 1);
        if (!no_pair && conv_pair96_supported(op0.cin, op0.cout, op0.ks, max_halo)) {
          GL.pair = true;
          // TMA-staged epilogue for launches with a residual / second output when its two tile buffers fit
          // (not for dilated windows: one buffer serialises the residual load behind the previous store
          // and measured slower than direct stores); otherwise the direct-store epilogue
          const bool staged = (L.flags & 3) != 0 && conv_pair96_stages(win_alloc, true) > 0;
          if (staged) L.flags |= kPairStaged;
          if (relu_in) L.flags |= kPairReluIn;
          L.stages = conv_pair96_stages(win_alloc, staged);
          for (size_t gi = 0; gi < grp.size(); ++gi) {
            const TcOp& op = p.tc[static_cast<size_t>(grp[gi])];
            TcGroup& g = L.g[gi];
            conv_tc_make_maps(plane_ptr(op.res_plane), ws.geo.Nalloc, op.cout, 128, g.pres);
            conv_tc_make_maps(plane_ptr(op.out_plane), ws.geo.Nalloc, op.cout, 128, g.pout);
            conv_tc_make_maps(plane_ptr(op.out2_plane), ws.geo.Nalloc, op.cout, 128, g.pout2);
          }
          ws.launches.push_back(GL);
          continue;
        }
        if (relu_in)
          throw Error(CNRX_ERR_UNSUPPORTED, "96-channel ReLU-on-load conv does not fit the CTA-pair kernel at this grid "
                                            "(plan option relu_on_load = 0 selects pre-activated planes)");
        int stages = 4;
        while (stages > 1 && conv_tc_smem_bytes(op0.cin, op0.cout, op0.ks, stages, win_alloc, L.flags) > 227 * 1024)
          --stages;
        if (conv_tc_smem_bytes(op0.cin, op0.cout, op0.ks, stages, win_alloc, L.flags) > 227 * 1024)
          throw Error(CNRX_ERR_UNSUPPORTED, "tcgen05 conv working set exceeds shared memory");
        L.stages = stages;
      }
      ws.launches.push_back(GL);
    }
}

void run_f32(cnrx_plan& p, const float* x, float* out, cudaStream_t s) {
  Workspace& ws = p.ws;
  auto val_ptr = [&](int v) -> float* {
    if (v == p.f32_in_val) return const_cast<float*>(x);
    if (v == p.f32_out_val) return out;
    return static_cast<float*>(ws.buffers[static_cast<size_t>(p.f32_val_buffer[static_cast<size_t>(v)])]);
  };
  const int B = ws.B, T = ws.T, F = ws.F;
  const int64_t rows = static_cast<int64_t>(B) * T * F;
  for (const auto& st : p.f32) {
    float* y = val_ptr(st.out_val);
    const float* a = val_ptr(st.in0);
    switch (st.kind) {
      case F_CONV: {
        ConvF32 c = st.conv;
        c.x = a;
        c.y = y;
        c.B = B;
        c.T = T;
        c.F = F;
        c.other = st.in1 >= 0 ? val_ptr(st.in1) : nullptr;
        p.note(launch_conv_f32(c, s), s, 2ll * c.kh * c.kw * c.cin * c.cout);
        break;
      }
      case F_DWCONV:
        p.note(launch_dwconv_f32(a, st.w, st.bias, y, B, T, F, st.C, st.kh, st.kw, s), s, 2ll * st.kh * st.kw * st.C);
        break;
      case F_AFFINE:
        p.note(launch_affine_f32(a, st.s, st.t, st.relu, y, rows, st.C, s), s);
        break;
      case F_RELU:
        p.note(launch_relu_f32(a, y, rows * st.C, s), s);
        break;
      case F_BINARY:
        p.note(launch_binary_f32(st.op, a, val_ptr(st.in1), y, rows * st.C, s), s);
        break;
      case F_LN:
        p.note(launch_layernorm_f32(a, st.g, st.b, y, rows, st.C, kLnEps, s), s);
        break;
      case F_CONCAT:
        p.note(launch_concat_f32(a, st.C, val_ptr(st.in1), st.C2, y, rows, s), s);
        break;
    }
  }
}

// input_kind: 0 = features [B,T,F,C] fp32, 1 = received grid y [B,T,F,N] complex
void trace_window(const unsigned long long* h) {
  const double span_us = (h[14] - ~h[13]) * 1e-3;
  const double mhz = h[15] ? static_cast<double>(h[kTraceTotal]) / static_cast<double>(h[15]) * 1e3 : 0.0;
  fprintf(stderr, "[trace]   CTAs %llu, MMA-loop span %.1f us, effective SM clock %.0f MHz\n", h[12], span_us, mhz);
}

void run_bf16(cnrx_plan& p, const float* in, int input_kind, int N, float* out, cudaStream_t s) {
  Workspace& ws = p.ws;
  auto plane_ptr = [&](int pl) {
    return static_cast<__nv_bfloat16*>(ws.buffers[static_cast<size_t>(p.planes[static_cast<size_t>(pl)].buffer)]);
  };
  if (p.need_plane0 && p.split) {
    // split plans: features in fp32 (reference layout: the caller's tensor, or featurized into the
    // workspace's fp32 buffer), then one pass into the (hi, lo) input plane
    const float* x = in;
    if (input_kind == 1) {
      float* feat = static_cast<float*>(ws.feat_buf);
      p.note(launch_featurize_ref(in, ws.geo, N, p.pt, feat, s), s);
      x = feat;
    }
    p.note(launch_pack_plane(x, ws.geo, p.in_ch, plane_ptr(0), p.planes[0].C, p.fp16, s, true), s);
  } else if (p.need_plane0) {
    __nv_bfloat16* in_plane = plane_ptr(0);
    if (input_kind == 0)
      p.note(launch_pack_plane(in, ws.geo, p.in_ch, in_plane, p.planes[0].C, p.fp16, s), s);
    else
      p.note(launch_featurize_plane(in, ws.geo, N, p.pt, in_plane, p.planes[0].C, p.fp16, s), s);
  }
  if (!p.stem_ops.empty()) {
    StemLaunch SL;
    std::memset(&SL, 0, sizeof(SL));
    SL.nops = static_cast<int>(p.stem_ops.size());
    SL.cin = p.tc[static_cast<size_t>(p.stem_ops[0])].cin_real;
    SL.N = N;
    SL.mode = input_kind;
    SL.fp16 = p.fp16;
    SL.x = input_kind == 0 ? in : nullptr;
    SL.y = input_kind == 1 ? in : nullptr;
    SL.pt = p.pt;
    int64_t fl = 0;
    for (int i = 0; i < SL.nops; ++i) {
      const TcOp& op = p.tc[static_cast<size_t>(p.stem_ops[static_cast<size_t>(i)])];
      StemOp& so = SL.op[i];
      so.w = op.stem_w;
      so.bias = op.bias;
      so.out = plane_ptr(op.out_plane);
      so.out2 = op.out2_plane >= 0 ? plane_ptr(op.out2_plane) : nullptr;
      so.s2 = op.s2;
      so.t2 = op.t2;
      so.cout = op.cout_real;
      so.relu = op.relu;
      fl += 2ll * op.cin_real * op.cout_real;
    }
    p.note(launch_stem(SL, ws.geo, s), s, fl);
  }
  size_t li = 0;
  for (int lv = 0; lv < p.n_levels; ++lv) {
    for (size_t gi = 0; gi < p.tc_groups_by_level[static_cast<size_t>(lv)].size(); ++gi) {
      const auto& grp = p.tc_groups_by_level[static_cast<size_t>(lv)][gi];
      if (grp.empty()) continue;
      const TcOp& op0 = p.tc[static_cast<size_t>(grp[0])];
      int64_t fl = 0;
      Workspace::GroupLaunch& GL = ws.launches[li++];
      if (GL.skip) continue;
      for (int k : grp) {
        const TcOp& o = p.tc[static_cast<size_t>(k)];
        fl += 2ll * o.ks * o.ks * o.cin_real * o.cout_real;
        if (GL.blk) {
          const TcOp& o1 = p.tc[static_cast<size_t>(o.blk_c1)];
          fl += 2ll * o1.ks * o1.ks * o1.cin_real * o1.cout_real;
        }
      }
      static const bool trace = getenv("CNRX_TRACE") != nullptr;
      static unsigned long long* dtrace = nullptr;
      if (GL.blk) {
        if (trace) {
          if (!dtrace) CNRX_CUDA(cudaMalloc(&dtrace, 32 * sizeof(unsigned long long)));
          CNRX_CUDA(cudaMemsetAsync(dtrace, 0, 32 * sizeof(unsigned long long), s));
          GL.blkl.trace = dtrace;
        }
        if (!GL.chain.empty()) {
          const PwProgram& hp = p.pw[static_cast<size_t>(p.hb_pw)].prog;
          for (size_t k = 0; k < GL.chain.size(); ++k) {
            BlkLaunch& C = GL.chain[k];
            C.fold.llr = out;
            const int64_t flc = fl / static_cast<int64_t>(GL.chain.size()) +
                                (C.epi == 2 ? 2ll * hp.C * hp.head_bits : 0);
            p.note(conv_blk64_launch(C, p.num_sms, s), s, flc);
          }
          continue;
        }
        p.note(conv_blk64_launch(GL.blkl, p.num_sms, s), s, fl);
        if (trace) {
          unsigned long long h[kBlkTraceSlots];
          CNRX_CUDA(cudaMemcpyAsync(h, dtrace, sizeof h, cudaMemcpyDeviceToHost, s));
          CNRX_CUDA(cudaStreamSynchronize(s));
          const double nt = static_cast<double>(h[kBlkTraceTiles] ? h[kBlkTraceTiles] : 1);
          fprintf(stderr,
                  "[trace] conv_blk64 relu_in=%d tiles=%llu per-tile cycles: prod_wait %.0f | mma1 wait_in %.0f wait_acc %.0f | "
                  "mma2 wait_in %.0f wait_acc %.0f | epi1 wait_full %.0f wait_w %.0f | epi2 wait_full %.0f | relu_wait %.0f | "
                  "total/tile %.0f\n",
                  GL.blkl.relu_in, h[kBlkTraceTiles], h[kBlkTraceProd] / nt, h[kBlkTraceM1In] / nt, h[kBlkTraceM1Acc] / nt,
                  h[kBlkTraceM2In] / nt, h[kBlkTraceM2Acc] / nt, h[kBlkTraceE1Full] / nt, h[kBlkTraceE1W] / nt,
                  h[kBlkTraceE2Full] / nt, h[kBlkTraceRelu] / nt, h[kBlkTraceTotal] / nt);
          fprintf(stderr, "[trace]   epi1 drain %.0f combine %.0f store %.0f (fence %.0f) | epi2 drain %.0f combine %.0f store %.0f\n",
                  h[kBlkTraceE1Drain] / nt, h[kBlkTraceE1Comb] / nt, h[kBlkTraceE1Store] / nt, h[kBlkTraceE1Fence] / nt, h[kBlkTraceE2Drain] / nt,
                  h[kBlkTraceE2Comb] / nt, h[kBlkTraceE2Store] / nt);
          fprintf(stderr, "[trace]   CTAs %llu, span %.1f us, effective SM clock %.0f MHz\n", h[12], (h[14] - ~h[13]) * 1e-3,
                  h[15] ? static_cast<double>(h[kBlkTraceTotal]) / static_cast<double>(h[15]) * 1e3 : 0.0);
          unsigned long long hx[32];
          CNRX_CUDA(cudaMemcpy(hx, dtrace, sizeof hx, cudaMemcpyDeviceToHost));
          const double e0 = static_cast<double>(~hx[24]);
          fprintf(stderr, "[trace]   phases from the first CTA entry: prologues done %.2f us | MMA loops %.2f .. %.2f us | "
                  "last exit %.2f us\n", (hx[25] - e0) * 1e-3, (~hx[13] - e0) * 1e-3, (hx[14] - e0) * 1e-3,
                  (hx[26] - e0) * 1e-3);
        }
        continue;
      }
      if (GL.ws) {
        if (trace) {
          if (!dtrace) CNRX_CUDA(cudaMalloc(&dtrace, 32 * sizeof(unsigned long long)));
          CNRX_CUDA(cudaMemsetAsync(dtrace, 0, 32 * sizeof(unsigned long long), s));
          GL.wsl.trace = dtrace;
        }
        static const int ws_debug = getenv("CNRX_WS_DEBUG") ? atoi(getenv("CNRX_WS_DEBUG")) : 0;
        GL.wsl.debug = ws_debug;
        if (GL.wsl.head_on) {
          GL.wsl.head.llr = out;
          const PwProgram& hp = p.pw[static_cast<size_t>(p.hf_pw)].prog;
          fl += 2ll * hp.C * hp.head_bits;
        }
        p.note(conv_ws64_launch(GL.wsl, p.num_sms, s), s, fl);
        if (trace) {
          unsigned long long h[kWsTraceSlots];
          CNRX_CUDA(cudaMemcpyAsync(h, dtrace, sizeof h, cudaMemcpyDeviceToHost, s));
          CNRX_CUDA(cudaStreamSynchronize(s));
          const double nt = static_cast<double>(h[kTraceTiles] ? h[kTraceTiles] : 1);
          fprintf(stderr, "[trace] conv_ws64 MMA loop-back %.0f commit %.0f cycles/tile\n", h[kWsTraceLoop] / nt,
                  h[kWsTraceCommit] / nt);
          fprintf(stderr,
                  "[trace] conv_ws64 tiles=%llu per-tile cycles: prod_wait %.0f mma_wait_full %.0f mma_wait_tmem %.0f "
                  "mma_issue %.0f | epi_wait %.0f combine %.0f stage_wait %.0f write %.0f | total/tile %.0f\n",
                  h[kTraceTiles], h[kTraceProdWaitEmpty] / nt, h[kTraceMmaWaitFull] / nt, h[kTraceMmaWaitTmem] / nt,
                  h[kTraceMmaIssue] / nt, h[kTraceEpiWaitFull] / nt, h[kWsTraceCombine] / nt,
                  h[kWsTraceStageWait] / nt, h[kWsTraceWrite] / nt, h[kTraceTotal] / nt);
          trace_window(h);
        }
        continue;
      }
      if (trace) {
        if (!dtrace) CNRX_CUDA(cudaMalloc(&dtrace, 32 * sizeof(unsigned long long)));
        CNRX_CUDA(cudaMemsetAsync(dtrace, 0, 32 * sizeof(unsigned long long), s));
        GL.tc.trace = dtrace;
      }
      if (GL.pair) {
        p.note(conv_pair96_launch(GL.tc, p.num_sms, s), s, fl);
        continue;
      }
      if (op0.llr_head) {  // 3x3 LLR head: the epilogue writes this forward's output
        GL.tc.g[0].llr = out;
        GL.x3l.g[0].llr = out;
      }
      if (GL.x3) {
        GL.x3l.trace = trace ? dtrace : nullptr;
        p.note(conv_x3_launch(op0.cin, op0.cout, op0.ks, GL.x3l, p.num_sms, s), s, fl);
        if (trace) {
          unsigned long long h[16];
          CNRX_CUDA(cudaMemcpyAsync(h, dtrace, sizeof h, cudaMemcpyDeviceToHost, s));
          CNRX_CUDA(cudaStreamSynchronize(s));
          const double nct = static_cast<double>(h[kTraceTiles] ? h[kTraceTiles] : 1);
          fprintf(stderr,
                  "[trace] %s tiles=%llu per-tile cycles: prod_wait_empty %.0f mma_wait_full %.0f mma_wait_tmem %.0f "
                  "mma_issue %.0f | epi(warp 3) wait %.0f work %.0f | mma-thread total/tile %.0f\n",
                  p.launch_names.back().c_str(), h[kTraceTiles], h[kTraceProdWaitEmpty] / nct, h[kTraceMmaWaitFull] / nct,
                  h[kTraceMmaWaitTmem] / nct, h[kTraceMmaIssue] / nct, h[kTraceEpiWaitFull] / nct, h[kTraceEpiWork] / nct,
                  h[kTraceTotal] / nct);
          trace_window(h);
        }
        continue;
      }
      p.note(conv_tc_launch(op0.cin, op0.cout, op0.ks, GL.tc, p.num_sms, s), s, fl);
      if (trace) {
        unsigned long long h[16];
        CNRX_CUDA(cudaMemcpyAsync(h, dtrace, sizeof h, cudaMemcpyDeviceToHost, s));
        CNRX_CUDA(cudaStreamSynchronize(s));
        const double nct = static_cast<double>(h[kTraceTiles] ? h[kTraceTiles] : 1);
        fprintf(stderr,
                "[trace] %s tiles=%llu per-tile cycles: prod_wait_empty %.0f mma_wait_full %.0f mma_wait_tmem %.0f "
                "mma_issue %.0f epi_wait %.0f epi_work %.0f | mma-thread total/tile %.0f\n",
                p.launch_names.back().c_str(), h[kTraceTiles], h[kTraceProdWaitEmpty] / nct,
                h[kTraceMmaWaitFull] / nct, h[kTraceMmaWaitTmem] / nct, h[kTraceMmaIssue] / nct,
                h[kTraceEpiWaitFull] / nct, h[kTraceEpiWork] / nct, h[kTraceTotal] / nct);
        trace_window(h);
      }
    }
    for (int k : p.pw_by_level[static_cast<size_t>(lv)]) {
      if (ws.head_fused && k == p.hf_pw) continue;      // ran in the last convs' epilogue
      if (ws.head_blk_fused && k == p.hb_pw) continue;  // ran in the last fused blocks' epilogues
      PwStep& st = p.pw[static_cast<size_t>(k)];
      if (st.dw) {
        p.note(launch_dwconv_plane(plane_ptr(st.plane_ids[0]), plane_ptr(st.out_plane), st.dw_w, st.dw_b, st.prog.C,
                                   st.dw_kh, st.dw_kw, st.dw_dil, p.fp16, p.split, ws.geo, s),
               s, 2ll * st.dw_kh * st.dw_kw * st.prog.C);
        continue;
      }
      if (st.concat) {
        const int ca = p.planes[static_cast<size_t>(st.plane_ids[0])].C;
        p.note(launch_concat_planes(plane_ptr(st.plane_ids[0]), ca, plane_ptr(st.plane_ids[1]), st.prog.C - ca,
                                    plane_ptr(st.out_plane), p.split, ws.geo, s),
               s);
        continue;
      }
      PwProgram prog = st.prog;
      prog.fp16 = p.fp16;
      prog.split = p.split;
      for (int j = 0; j < st.n_planes; ++j) prog.planes[j] = plane_ptr(st.plane_ids[j]);
      if (st.out_plane >= 0)
        prog.out_plane = plane_ptr(st.out_plane);
      else
        prog.llr = out;
      prog.out2_plane = st.out2_plane >= 0 ? plane_ptr(st.out2_plane) : nullptr;
      p.note(launch_pw_program(prog, ws.geo, s), s);
    }
  }
}

void check_shape(cnrx_plan& p, int64_t B, int64_t T, int64_t F, int64_t C) {
  require(B > 0 && T > 0 && F > 0 && C > 0, "tensor dimensions must be positive");
  require(C == p.in_ch, "network expects " + std::to_string(p.in_ch) + " input channels, got [" + std::to_string(B) +
                            "," + std::to_string(T) + "," + std::to_string(F) + "," + std::to_string(C) + "]");
  require(B < (1ll << 31) && T < 4096 && F < (1 << 20), "tensor dimensions too large");
}

void* ensure_dev(Workspace& ws, void*& buf, size_t& cap, size_t bytes) {
  if (cap < bytes) {
    ws_free(ws, buf);
    buf = nullptr;  // a failed cudaMalloc must not leave a stale pointer / capacity behind
    cap = 0;
    buf = ws_malloc(ws, bytes);
    cap = bytes;
  }
  return buf;
}

// Slots per forward whose workspace (activation planes, or fp32 node buffers, plus the fp32 feature
// buffer) fits the plan's memory budget (55 % of the device's HBM): bigger batches run as consecutive
// slot chunks through the same workspace (every op is per slot, so the LLRs are the same).
int64_t max_batch(const cnrx_plan& p, int64_t T, int64_t F) {
  if (p.mem_budget == 0) return int64_t{1} << 40;
  double per_slot = static_cast<double>(T * F * p.in_ch) * sizeof(float);  // fp32 features (receive path)
  if (p.precision == CNRX_FP32) {
    for (int c : p.f32_buf_channels) per_slot += static_cast<double>(T * F * c) * sizeof(float);
  } else {
    const double rows = static_cast<double>(F + p.npad) * static_cast<double>(T + 1);
    for (int c : p.buf_channels) per_slot += rows * c * 2.0 * (p.split ? 2 : 1);
  }
  return std::max<int64_t>(1, static_cast<int64_t>(static_cast<double>(p.mem_budget) / per_slot));
}

void run_forward(cnrx_plan& p, const float* x_dev, int64_t B, int64_t T, int64_t F, float* out_dev, int input_kind,
                 int N, cudaStream_t s) {
  const int64_t cap = max_batch(p, T, F);
  if (B > cap) {
    const int64_t in_slot = T * F * (input_kind == 1 ? 2 * N : p.in_ch), out_slot = T * F * p.out_ch;
    for (int64_t b0 = 0; b0 < B; b0 += cap)
      run_forward(p, x_dev + b0 * in_slot, std::min(cap, B - b0), T, F, out_dev + b0 * out_slot, input_kind, N, s);
    return;
  }
  ensure_workspace(p, static_cast<int>(B), static_cast<int>(T), static_cast<int>(F));
  float* feat = nullptr;  // fp32 plans on the receive path: features in the reference layout
  if ((p.precision == CNRX_FP32 || p.split) && input_kind == 1) {  // allocated outside any graph capture
    const size_t bytes = static_cast<size_t>(B * T * F * p.in_ch) * sizeof(float);
    feat = static_cast<float*>(ensure_dev(p.ws, p.ws.feat_buf, p.ws.feat_bytes, bytes));
  }
  auto enqueue = [&]() {
    p.launch_names.clear();
    p.launch_flops.clear();
    if (p.profile && !p.capture) {
      p.prof_events.emplace_back();
      cudaEvent_t e = p.take_event();
      CNRX_CUDA(cudaEventRecord(e, s));
      p.prof_events.back().push_back(e);
    }
    if (p.precision == CNRX_FP32) {
      if (input_kind == 1) {
        // featurize into an fp32 reference-layout buffer, then run the node program on it
        PlaneGeom g = make_geom(static_cast<int>(B), static_cast<int>(T), static_cast<int>(F), 1);
        p.note(launch_featurize_ref(x_dev, g, N, p.pt, feat, s), s);
        run_f32(p, feat, out_dev, s);
      } else {
        run_f32(p, x_dev, out_dev, s);
      }
    } else {
      run_bf16(p, x_dev, input_kind, N, out_dev, s);
    }
  };
  // The workspace planes are shared by every call of this plan: a call on a different stream than the
  // previous one first waits for that call's kernels (calls on one stream are ordered already).
  auto order_in = [&](cudaStream_t st) {
    if (p.ws_used && p.ws_stream != st) CNRX_CUDA(cudaStreamWaitEvent(st, p.ws_done, 0));
  };
  auto order_out = [&](cudaStream_t st) {
    if (!p.ws_done) CNRX_CUDA(cudaEventCreateWithFlags(&p.ws_done, cudaEventDisableTiming));
    CNRX_CUDA(cudaEventRecord(p.ws_done, st));
    p.ws_stream = st;
    p.ws_used = true;
  };
  if (!p.capture) {
    order_in(s);
    enqueue();
    order_out(s);
    return;
  }
  // A legacy / per-thread default stream cannot be captured: capture and replay on the plan's own
  // stream, ordered after and before the caller's stream with events.
  cudaStream_t caller = s;
  const bool fence = s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread;
  if (fence) {
    s = p.stream;
    if (!p.fence_in) {
      CNRX_CUDA(cudaEventCreateWithFlags(&p.fence_in, cudaEventDisableTiming));
      CNRX_CUDA(cudaEventCreateWithFlags(&p.fence_out, cudaEventDisableTiming));
    }
    CNRX_CUDA(cudaEventRecord(p.fence_in, caller));
    CNRX_CUDA(cudaStreamWaitEvent(s, p.fence_in, 0));
  }
  char key[256];
  snprintf(key, sizeof key, "%p/%p/%lld/%lld/%lld/%d/%p", static_cast<const void*>(x_dev), static_cast<void*>(out_dev),
           static_cast<long long>(B), static_cast<long long>(T), static_cast<long long>(F), input_kind,
           static_cast<void*>(s));
  if (!p.gexec || p.gkey != key) {
    if (p.gexec) {
      cudaGraphExecDestroy(p.gexec);
      p.gexec = nullptr;
    }
    cudaGraph_t graph;
    CNRX_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(s, &graph);
      throw;
    }
    CNRX_CUDA(cudaStreamEndCapture(s, &graph));
    CNRX_CUDA(cudaGraphInstantiate(&p.gexec, graph, 0));
    cudaGraphDestroy(graph);
    p.gkey = key;
  }
  order_in(s);
  CNRX_CUDA(cudaGraphLaunch(p.gexec, s));
  order_out(s);
  if (fence) {
    CNRX_CUDA(cudaEventRecord(p.fence_out, s));
    CNRX_CUDA(cudaStreamWaitEvent(caller, p.fence_out, 0));
  }
}


void build_pilot_tables(cnrx_plan& p, int64_t T, int64_t F, const float* pilots, const uint8_t* mask) {
  std::vector<int> syms;
  for (int64_t t = 0; t < T; ++t) {
    bool any = false;
    for (int64_t f = 0; f < F; ++f) any |= mask[t * F + f] != 0;
    if (any) syms.push_back(static_cast<int>(t));
  }
  require(!syms.empty(), "pilot pattern has no pilots");
  if (static_cast<int>(syms.size()) > kMaxPilotSyms) throw Error(CNRX_ERR_UNSUPPORTED, "more than 8 pilot symbols");
  const int ns = static_cast<int>(syms.size());
  std::vector<int32_t> flo(static_cast<size_t>(ns * F)), fhi(static_cast<size_t>(ns * F));
  std::vector<float> wf(static_cast<size_t>(ns * F));
  std::vector<float> x(static_cast<size_t>(2 * T * F), 0.f), inv(static_cast<size_t>(2 * T * F), 0.f);
  for (int64_t i = 0; i < T * F; ++i)
    if (mask[i]) {
      const double xr = pilots[2 * i], xi = pilots[2 * i + 1];
      const double den = xr * xr + xi * xi;
      require(den > 0, "zero pilot symbol");
      x[static_cast<size_t>(2 * i)] = static_cast<float>(xr);
      x[static_cast<size_t>(2 * i + 1)] = static_cast<float>(xi);
      inv[static_cast<size_t>(2 * i)] = static_cast<float>(xr / den);
      inv[static_cast<size_t>(2 * i + 1)] = static_cast<float>(-xi / den);
    }
  for (int j = 0; j < ns; ++j) {
    std::vector<int> pf;
    for (int64_t f = 0; f < F; ++f)
      if (mask[syms[static_cast<size_t>(j)] * F + f]) pf.push_back(static_cast<int>(f));
    for (int64_t f = 0; f < F; ++f) {
      int k0, k1;
      double w;
      if (f <= pf.front()) {
        k0 = k1 = 0;
        w = 0;
      } else if (f >= pf.back()) {
        k0 = k1 = static_cast<int>(pf.size()) - 1;
        w = 0;
      } else {
        k0 = 0;
        while (pf[static_cast<size_t>(k0 + 1)] < f) ++k0;
        k1 = k0 + 1;
        w = static_cast<double>(f - pf[static_cast<size_t>(k0)]) / (pf[static_cast<size_t>(k1)] - pf[static_cast<size_t>(k0)]);
      }
      flo[static_cast<size_t>(j * F + f)] = pf[static_cast<size_t>(k0)];
      fhi[static_cast<size_t>(j * F + f)] = pf[static_cast<size_t>(k1)];
      wf[static_cast<size_t>(j * F + f)] = static_cast<float>(w);
    }
  }
  std::vector<int32_t> jlo(static_cast<size_t>(T)), jhi(static_cast<size_t>(T));
  std::vector<float> wt(static_cast<size_t>(T));
  for (int64_t t = 0; t < T; ++t) {
    int j0, j1;
    double w;
    if (t <= syms.front()) {
      j0 = j1 = 0;
      w = 0;
    } else if (t >= syms.back()) {
      j0 = j1 = ns - 1;
      w = 0;
    } else {
      j0 = 0;
      while (syms[static_cast<size_t>(j0 + 1)] < t) ++j0;
      j1 = j0 + 1;
      w = static_cast<double>(t - syms[static_cast<size_t>(j0)]) / (syms[static_cast<size_t>(j1)] - syms[static_cast<size_t>(j0)]);
    }
    jlo[static_cast<size_t>(t)] = j0;
    jhi[static_cast<size_t>(t)] = j1;
    wt[static_cast<size_t>(t)] = static_cast<float>(w);
  }
  PilotTablesDev pt{};
  pt.n_sym = ns;
  for (int j = 0; j < ns; ++j) pt.sym[j] = syms[static_cast<size_t>(j)];
  pt.flo = static_cast<const int32_t*>(p.upload_bytes(flo.data(), flo.size() * 4));
  pt.fhi = static_cast<const int32_t*>(p.upload_bytes(fhi.data(), fhi.size() * 4));
  pt.wf = p.upload(wf);
  pt.jlo = static_cast<const int32_t*>(p.upload_bytes(jlo.data(), jlo.size() * 4));
  pt.jhi = static_cast<const int32_t*>(p.upload_bytes(jhi.data(), jhi.size() * 4));
  pt.wt = p.upload(wt);
  pt.x = p.upload(x);
  pt.inv_x = p.upload(inv);
  p.pt = pt;
  p.pT = static_cast<int>(T);
  p.pF = static_cast<int>(F);
  p.has_pilots = true;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CNRX_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

namespace {

// Host-buffer entry points: the slot batch is cut into chunks so that the host->device copy of chunk
// k+1 and the device->host copy of chunk k-1 run on the copy engines while chunk k computes (full
// overlap needs page-locked host buffers; pageable ones still give correct results).  Slots are
// independent, so chunking changes nothing in the results.
int pipeline_chunks(const cnrx_plan& p, int64_t B) {
  if (p.capture) return 1;  // a captured graph is keyed on its pointers: keep one launch
  if (p.opt.pipeline_chunks >= 1) return static_cast<int>(std::min<int64_t>(p.opt.pipeline_chunks, B));
  // measured on cfg2 (B=256): 3-4 chunks maximise e2e; more chunks pay each launch's fixed cost again
  return static_cast<int>(std::min<int64_t>(4, std::max<int64_t>(1, B / 48)));
}

template <class Run>
void host_pipeline(cnrx_plan& p, const float* in, size_t in_per_slot, float* out, size_t out_per_slot, int64_t B,
                   Run&& run) {
  const size_t in_bytes = static_cast<size_t>(B) * in_per_slot;
  const size_t out_bytes = static_cast<size_t>(B) * out_per_slot;
  char* din = static_cast<char*>(ensure_dev(p.ws, p.ws.in_buf, p.ws.in_bytes, in_bytes));
  char* dout = static_cast<char*>(ensure_dev(p.ws, p.ws.out_buf, p.ws.out_bytes, out_bytes));
  const int n = pipeline_chunks(p, B);
  if (n == 1) {
    CNRX_CUDA(cudaMemcpyAsync(din, in, in_bytes, cudaMemcpyHostToDevice, p.stream));
    run(reinterpret_cast<const float*>(din), B, reinterpret_cast<float*>(dout), p.stream);
    CNRX_CUDA(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, p.stream));
    CNRX_CUDA(cudaStreamSynchronize(p.stream));
    return;
  }
  if (!p.h2d) {
    CNRX_CUDA(cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking));
    CNRX_CUDA(cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking));
  }
  while (p.pipe_ev.size() < static_cast<size_t>(2 * n)) {
    cudaEvent_t e;
    CNRX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p.pipe_ev.push_back(e);
  }
  // the previous call's work on the plan stream (and its buffers) is finished before we return, but
  // order the copy streams after anything the caller queued on the plan stream anyway
  CNRX_CUDA(cudaEventRecord(p.pipe_ev[0], p.stream));
  CNRX_CUDA(cudaStreamWaitEvent(p.h2d, p.pipe_ev[0], 0));
  // tapered chunks (first and last 1/8 of a middle chunk; measured e2e +1.5 % over half-size): the first upload and the last download are the only
  // copies not hidden behind a chunk's kernels
  // CNRX_PIPELINE_TAPER: size of the first / last chunk relative to the others (0 or 1: no taper)
  const double tw = p.opt.pipeline_taper;
  const bool taper = tw > 0.0 && tw < 1.0;
  std::vector<int64_t> bounds(static_cast<size_t>(n) + 1, 0);
  const double units = taper && n > 2 ? n - 2.0 + 2.0 * tw : static_cast<double>(n);
  double acc = 0;
  for (int k = 0; k < n; ++k) {
    acc += (taper && n > 2 && (k == 0 || k == n - 1)) ? tw : 1.0;
    bounds[static_cast<size_t>(k) + 1] = std::min<int64_t>(B, static_cast<int64_t>(std::llround(acc / units * B)));
  }
  bounds[static_cast<size_t>(n)] = B;
  for (int k = 0; k < n; ++k) {
    const int64_t b0 = bounds[static_cast<size_t>(k)], nb = bounds[static_cast<size_t>(k) + 1] - b0;
    if (nb <= 0) continue;
    cudaEvent_t landed = p.pipe_ev[static_cast<size_t>(2 * k)], done = p.pipe_ev[static_cast<size_t>(2 * k + 1)];
    CNRX_CUDA(cudaMemcpyAsync(din + b0 * in_per_slot, reinterpret_cast<const char*>(in) + b0 * in_per_slot,
                              static_cast<size_t>(nb) * in_per_slot, cudaMemcpyHostToDevice, p.h2d));
    CNRX_CUDA(cudaEventRecord(landed, p.h2d));
    CNRX_CUDA(cudaStreamWaitEvent(p.stream, landed, 0));
    run(reinterpret_cast<const float*>(din + b0 * in_per_slot), nb, reinterpret_cast<float*>(dout + b0 * out_per_slot),
        p.stream);
    CNRX_CUDA(cudaEventRecord(done, p.stream));
    CNRX_CUDA(cudaStreamWaitEvent(p.d2h, done, 0));
    CNRX_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(out) + b0 * out_per_slot, dout + b0 * out_per_slot,
                              static_cast<size_t>(nb) * out_per_slot, cudaMemcpyDeviceToHost, p.d2h));
  }
  CNRX_CUDA(cudaStreamSynchronize(p.d2h));
  CNRX_CUDA(cudaStreamSynchronize(p.stream));
}

}  // namespace

// ================================================================================================
// C ABI
// ================================================================================================
namespace {
// contiguous slot ranges, one host thread per plan (no collective on the data path)
template <class Call>
int run_sharded(cnrx_plan* const* plans, int32_t n_plans, int64_t B, Call&& call) {
  if (!plans || n_plans < 1) return fail(CNRX_ERR_INVALID_ARGUMENT, "no plans");
  const int64_t per = (B + n_plans - 1) / n_plans;
  std::vector<int> rcs(static_cast<size_t>(n_plans), CNRX_OK);
  std::vector<std::string> msgs(static_cast<size_t>(n_plans));
  std::vector<std::thread> th;
  for (int i = 0; i < n_plans; ++i) {
    const int64_t b0 = i * per, b1 = std::min(B, b0 + per);
    if (b0 >= b1) break;
    th.emplace_back([&, i, b0, b1] {
      rcs[static_cast<size_t>(i)] = call(plans[i], b0, b1 - b0);
      if (rcs[static_cast<size_t>(i)] != CNRX_OK) msgs[static_cast<size_t>(i)] = cnrx_last_error();
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < n_plans; ++i)
    if (rcs[static_cast<size_t>(i)] != CNRX_OK)
      return fail(rcs[static_cast<size_t>(i)], "shard " + std::to_string(i) + ": " + msgs[static_cast<size_t>(i)]);
  return CNRX_OK;
}
}  // namespace

extern "C" {

const char* cnrx_last_error(void) { return g_last_error.c_str(); }

void cnrx_plan_options_default(cnrx_plan_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = static_cast<int32_t>(sizeof(*o));
  o->fused_blocks = 1;
  o->fused_head = 0;
  o->tensor_core_head = 0;
  o->cta_pair = 1;
  o->weights_stationary = 1;
  o->relu_on_load = 1;
  o->cuda_core_stem = 0;
  o->pipeline_chunks = 0;
  o->pipeline_taper = 0.125f;
}

namespace {
// A/B switches of cnrx_plan_create, read once per plan creation.
void apply_env_options(cnrx_plan_options* o) {
  auto env_int = [](const char* name, int* v) {
    const char* e = std::getenv(name);
    if (e) *v = std::atoi(e);
    return e != nullptr;
  };
  int v = 0;
  if (env_int("CNRX_BLK", &v)) o->fused_blocks = v != 0;
  if (std::getenv("CNRX_HEADFUSE")) o->fused_head = 1;
  if (std::getenv("CNRX_NO_HEADFUSE")) o->fused_head = 0;
  if (std::getenv("CNRX_TC_HEAD")) o->tensor_core_head = 1;
  if (std::getenv("CNRX_NO_TMA_HEAD")) o->tensor_core_head = 0;
  if (env_int("CNRX_NO_PAIR", &v) && v != 0) o->cta_pair = 0;
  if (std::getenv("CNRX_NO_WS")) o->weights_stationary = 0;
  if (std::getenv("CNRX_NO_RELU_IN")) o->relu_on_load = 0;
  if (std::getenv("CNRX_STEM")) o->cuda_core_stem = 1;
  if (env_int("CNRX_PIPELINE_CHUNKS", &v) && v >= 1) o->pipeline_chunks = v;
  if (const char* e = std::getenv("CNRX_PIPELINE_TAPER")) o->pipeline_taper = static_cast<float>(std::atof(e));
}
}  // namespace

int cnrx_plan_create(const cnrx_node* nodes, int32_t n_nodes, int32_t input_node, int32_t output_node,
                     const cnrx_param* params, int32_t n_params, const uint8_t* bn_ready, int32_t n_bn,
                     int32_t precision, int32_t device, cnrx_plan** out) {
  cnrx_plan_options o;
  cnrx_plan_options_default(&o);
  apply_env_options(&o);
  return cnrx_plan_create_ex(nodes, n_nodes, input_node, output_node, params, n_params, bn_ready, n_bn, precision,
                             device, &o, out);
}

int cnrx_get_plan_options(const cnrx_plan* plan, cnrx_plan_options* opt) {
  if (!plan || !opt) return fail(CNRX_ERR_INVALID_ARGUMENT, "null argument");
  *opt = plan->opt;
  return CNRX_OK;
}

int cnrx_plan_create_ex(const cnrx_node* nodes, int32_t n_nodes, int32_t input_node, int32_t output_node,
                        const cnrx_param* params, int32_t n_params, const uint8_t* bn_ready, int32_t n_bn,
                        int32_t precision, int32_t device, const cnrx_plan_options* options, cnrx_plan** out) {
  if (!out) return fail(CNRX_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  if (options && options->struct_size != static_cast<int32_t>(sizeof(cnrx_plan_options)))
    return fail(CNRX_ERR_INVALID_ARGUMENT, "cnrx_plan_options.struct_size mismatch (header / library version)");
  auto plan = std::make_unique<cnrx_plan>();
  if (options)
    plan->opt = *options;
  else
    cnrx_plan_options_default(&plan->opt);
  const int rc = guarded([&] {
    require(nodes && n_nodes > 0, "empty network");
    require(precision == CNRX_FP32 || precision == CNRX_BF16 || precision == CNRX_FP16 || precision == CNRX_BF16X3 ||
                precision == CNRX_FP16X3,
            "unknown precision");
    int ndev = 0;
    CNRX_CUDA(cudaGetDeviceCount(&ndev));
    require(device >= 0 && device < ndev, "no such CUDA device " + std::to_string(device));
    DeviceGuard dg(device);
    cudaDeviceProp prop;
    CNRX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (precision != CNRX_FP32 && prop.major != 10)
      throw Error(CNRX_ERR_UNSUPPORTED, "bf16 / fp16 tcgen05 plan needs an sm_100 (Blackwell) device");
    plan->precision = precision;
    plan->fp16 = precision == CNRX_FP16 || precision == CNRX_FP16X3;
    plan->split = precision == CNRX_BF16X3 || precision == CNRX_FP16X3;
    if (plan->split) {
      // split plans run every conv on conv_x3.cu and the tail on the generic pointwise programs
      plan->opt.fused_blocks = 0;
      plan->opt.fused_head = 0;
      plan->opt.tensor_core_head = 0;
      plan->opt.cta_pair = 0;
      plan->opt.weights_stationary = 0;
      plan->opt.cuda_core_stem = 0;
    }
    plan->device = device;
    plan->num_sms = prop.multiProcessorCount;
    plan->mem_budget = static_cast<size_t>(0.55 * static_cast<double>(prop.totalGlobalMem));
    if (const char* mb = std::getenv("CNRX_MEM_BUDGET_MB"))  // tests of the slot-chunked forward only
      plan->mem_budget = static_cast<size_t>(std::atof(mb) * 1048576.0);
    plan->nodes.assign(nodes, nodes + n_nodes);
    plan->in_node = input_node;
    plan->out_node = output_node;
    plan->params.resize(static_cast<size_t>(n_params));
    for (int i = 0; i < n_params; ++i) {
      HostParam& hp = plan->params[static_cast<size_t>(i)];
      hp.name = params[i].name ? params[i].name : "";
      require(params[i].rank >= 1 && params[i].rank <= 4, "parameter rank must be 1..4");
      hp.dims.assign(params[i].dims, params[i].dims + params[i].rank);
      hp.learnable = params[i].learnable != 0;
      const int64_t nel = hp.numel();
      require(nel > 0 && params[i].data, "parameter " + hp.name + " has no data");
      hp.data.assign(params[i].data, params[i].data + nel);
    }
    plan->bn_ready.assign(bn_ready, bn_ready + n_bn);
    validate_graph(*plan);
    CNRX_CUDA(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
    if (precision == CNRX_FP32)
      compile_f32(*plan);
    else
      Bf16Compiler(*plan).compile();
  });
  if (rc != CNRX_OK) {
    cnrx_plan_destroy(plan.release());
    return rc;
  }
  *out = plan.release();
  return CNRX_OK;
}

void cnrx_plan_destroy(cnrx_plan* plan) {
  if (!plan) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(plan->device);
  if (plan->stream) cudaStreamSynchronize(plan->stream);
  if (plan->gexec) cudaGraphExecDestroy(plan->gexec);
  if (plan->fence_in) cudaEventDestroy(plan->fence_in);
  if (plan->fence_out) cudaEventDestroy(plan->fence_out);
  for (void* b : plan->ws.buffers) ws_free(plan->ws, b);
  ws_free(plan->ws, plan->ws.in_buf);
  ws_free(plan->ws, plan->ws.out_buf);
  ws_free(plan->ws, plan->ws.feat_buf);
  ws_free(plan->ws, plan->ws.classic_buf);
  for (void* b : plan->ws.fold_bufs) ws_free(plan->ws, b);
  if (plan->classic_done) cudaEventDestroy(plan->classic_done);
  for (void* d : plan->dev_allocs) cudaFree(d);
  for (auto& evs : plan->prof_events)
    for (auto e : evs) cudaEventDestroy(e);
  for (auto e : plan->event_pool) cudaEventDestroy(e);
  for (auto e : plan->pipe_ev) cudaEventDestroy(e);
  if (plan->ws_done) cudaEventDestroy(plan->ws_done);
  if (plan->h2d) cudaStreamDestroy(plan->h2d);
  if (plan->d2h) cudaStreamDestroy(plan->d2h);
  if (plan->stream) cudaStreamDestroy(plan->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete plan;
}

// Drops every workspace buffer (plane / node buffers, staging, feature and fold buffers) so the next call
// reallocates them; a captured graph refers to the old addresses and goes with them.
static void release_workspace(cnrx_plan& p) {
  Workspace& ws = p.ws;
  if (p.gexec) {
    cudaGraphExecDestroy(p.gexec);
    p.gexec = nullptr;
    p.gkey.clear();
  }
  for (void* b : ws.buffers) ws_free(ws, b);
  ws.buffers.clear();
  ws.sizes.clear();
  ws.launches.clear();
  ws.cap_B = 0;
  ws.B = ws.T = ws.F = -1;
  for (void*& b : ws.fold_bufs) {
    ws_free(ws, b);
    b = nullptr;
  }
  ws.fold_bytes = 0;
  void** bufs[] = {&ws.in_buf, &ws.out_buf, &ws.feat_buf, &ws.classic_buf};
  size_t* caps[] = {&ws.in_bytes, &ws.out_bytes, &ws.feat_bytes, &ws.classic_bytes};
  for (int i = 0; i < 4; ++i) {
    ws_free(ws, *bufs[i]);
    *bufs[i] = nullptr;
    *caps[i] = 0;
  }
}

int cnrx_plan_set_guard_bands(cnrx_plan* plan, int32_t enable) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    DeviceGuard dg(plan->device);
    CNRX_CUDA(cudaDeviceSynchronize());
    release_workspace(*plan);
    plan->ws.guard = enable != 0;
  });
}

int cnrx_plan_check_guard_bands(cnrx_plan* plan, int64_t* n_buffers, int64_t* bad_bytes) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    require(n_buffers && bad_bytes, "null result pointer");
    require(plan->ws.guard, "guard bands are off (cnrx_plan_set_guard_bands)");
    DeviceGuard dg(plan->device);
    CNRX_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned char> h(kGuardBytes);
    int64_t bad = 0;
    for (const auto& gb : plan->ws.guarded)
      for (int side = 0; side < 2; ++side) {
        CNRX_CUDA(cudaMemcpy(h.data(), gb.base + (side ? kGuardBytes + gb.bytes : 0), kGuardBytes, cudaMemcpyDeviceToHost));
        for (unsigned char v : h) bad += v != kGuardByte;
      }
    *n_buffers = static_cast<int64_t>(plan->ws.guarded.size());
    *bad_bytes = bad;
  });
}

int cnrx_plan_guard_band_ptr(cnrx_plan* plan, int64_t index, int32_t side, void** band_dev) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    require(band_dev != nullptr, "null result pointer");
    require(index >= 0 && index < static_cast<int64_t>(plan->ws.guarded.size()) && (side == 0 || side == 1),
            "no such guard band");
    const auto& gb = plan->ws.guarded[static_cast<size_t>(index)];
    *band_dev = gb.base + (side ? kGuardBytes + gb.bytes : 0);
  });
}

int cnrx_forward_device(cnrx_plan* plan, const float* x_dev, int64_t B, int64_t T, int64_t F, int64_t C,
                        int32_t mode, float* out_dev, void* stream) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    if (mode != CNRX_MODE_EVAL)
      throw Error(CNRX_ERR_UNSUPPORTED, "only NormMode::eval is supported (train mutates running statistics)");
    check_shape(*plan, B, T, F, C);
    require(x_dev && out_dev, "null tensor pointer");
    DeviceGuard dg(plan->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : plan->stream;
    run_forward(*plan, x_dev, B, T, F, out_dev, 0, 0, s);
  });
}

int cnrx_forward(cnrx_plan* plan, const float* x, int64_t B, int64_t T, int64_t F, int64_t C, int32_t mode,
                 float* out) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    if (mode != CNRX_MODE_EVAL)
      throw Error(CNRX_ERR_UNSUPPORTED, "only NormMode::eval is supported (train mutates running statistics)");
    check_shape(*plan, B, T, F, C);
    require(x && out, "null tensor pointer");
    DeviceGuard dg(plan->device);
    host_pipeline(*plan, x, static_cast<size_t>(T * F * C) * sizeof(float), out,
                  static_cast<size_t>(T * F * plan->out_ch) * sizeof(float), B,
                  [&](const float* xi, int64_t nb, float* yo, cudaStream_t s) {
                    run_forward(*plan, xi, nb, T, F, yo, 0, 0, s);
                  });
  });
}

int cnrx_set_pilots(cnrx_plan* plan, int64_t T, int64_t F, const float* pilots, const uint8_t* mask) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    require(T > 0 && F > 0 && pilots && mask, "bad pilot grid");
    DeviceGuard dg(plan->device);
    build_pilot_tables(*plan, T, F, pilots, mask);
    if (plan->gexec) {
      cudaGraphExecDestroy(plan->gexec);
      plan->gexec = nullptr;
      plan->gkey.clear();
    }
  });
}

static void check_receive(cnrx_plan& p, int64_t B, int64_t T, int64_t F, int64_t N) {
  require(p.has_pilots, "cnrx_set_pilots must be called before receive");
  require(T == p.pT && F == p.pF, "received grid [T,F] does not match the pilot grid");
  require(N >= 1 && 6 * N == p.in_ch, "network expects " + std::to_string(p.in_ch) + " input channels, i.e. " +
                                          std::to_string(p.in_ch / 6) + " antennas, got N=" + std::to_string(N));
  require(B > 0, "tensor dimensions must be positive");
}

int cnrx_receive_device(cnrx_plan* plan, const float* y_dev, int64_t B, int64_t T, int64_t F, int64_t N,
                        float* llr_dev, void* stream) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    check_receive(*plan, B, T, F, N);
    require(y_dev && llr_dev, "null tensor pointer");
    DeviceGuard dg(plan->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : plan->stream;
    run_forward(*plan, y_dev, B, T, F, llr_dev, 1, static_cast<int>(N), s);
  });
}

int cnrx_receive(cnrx_plan* plan, const float* y, int64_t B, int64_t T, int64_t F, int64_t N, float* llr) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    check_receive(*plan, B, T, F, N);
    require(y && llr, "null tensor pointer");
    DeviceGuard dg(plan->device);
    host_pipeline(*plan, y, static_cast<size_t>(T * F * N) * 2 * sizeof(float), llr,
                  static_cast<size_t>(T * F * plan->out_ch) * sizeof(float), B,
                  [&](const float* yi, int64_t nb, float* lo, cudaStream_t s) {
                    run_forward(*plan, yi, nb, T, F, lo, 1, static_cast<int>(N), s);
                  });
  });
}

int cnrx_featurize_device(cnrx_plan* plan, const float* y_dev, int64_t B, int64_t T, int64_t F, int64_t N,
                          float* feat_dev, void* stream) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    require(plan->has_pilots, "cnrx_set_pilots must be called before featurize");
    require(T == plan->pT && F == plan->pF && B > 0 && N >= 1, "received grid does not match the pilot grid");
    DeviceGuard dg(plan->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : plan->stream;
    PlaneGeom g = make_geom(static_cast<int>(B), static_cast<int>(T), static_cast<int>(F), 1);
    launch_featurize_ref(y_dev, g, static_cast<int>(N), plan->pt, feat_dev, s);
  });
}


int cnrx_feature_plane_device(cnrx_plan* plan, const float* y_dev, int64_t B, int64_t T, int64_t F, int64_t N,
                              uint16_t* out_dev, int32_t* cpad) {
  if (!plan || !cpad) return fail(CNRX_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    if (plan->precision == CNRX_FP32 || plan->split)
      throw Error(CNRX_ERR_UNSUPPORTED, "fp32 and split-precision plans have no 16-bit feature plane");
    check_receive(*plan, B, T, F, N);
    DeviceGuard dg(plan->device);
    CNRX_CUDA(cudaDeviceSynchronize());  // test hook: fully ordered against any earlier call
    ensure_workspace(*plan, static_cast<int>(B), static_cast<int>(T), static_cast<int>(F));
    const Workspace& ws = plan->ws;
    auto* plane = static_cast<__nv_bfloat16*>(ws.buffers[static_cast<size_t>(plan->planes[0].buffer)]);
    *cpad = plan->planes[0].C;
    launch_featurize_plane(y_dev, ws.geo, static_cast<int>(N), plan->pt, plane, plan->planes[0].C, plan->fp16,
                           plan->stream);
    launch_plane_rows_to_ref(plane, ws.geo, plan->planes[0].C, out_dev, plan->stream);
    CNRX_CUDA(cudaStreamSynchronize(plan->stream));
  });
}

int cnrx_forward_sharded(cnrx_plan* const* plans, int32_t n_plans, const float* x, int64_t B, int64_t T, int64_t F,
                         int64_t C, int32_t mode, float* out) {
  return run_sharded(plans, n_plans, B, [&](cnrx_plan* p, int64_t b0, int64_t nb) {
    return cnrx_forward(p, x + b0 * T * F * C, nb, T, F, C, mode, out + b0 * T * F * p->out_ch);
  });
}

int cnrx_receive_sharded(cnrx_plan* const* plans, int32_t n_plans, const float* y, int64_t B, int64_t T, int64_t F,
                         int64_t N, float* llr) {
  return run_sharded(plans, n_plans, B, [&](cnrx_plan* p, int64_t b0, int64_t nb) {
    return cnrx_receive(p, y + b0 * T * F * N * 2, nb, T, F, N, llr + b0 * T * F * p->out_ch);
  });
}


int cnrx_generate_slots(const cnrx_link* link, int64_t B, uint64_t seed, uint64_t slot0, float* y_dev,
                        uint8_t* bits_dev, float* h_dev, void* stream) {
  return guarded([&] {
    require(link != nullptr, "null link");
    require(B > 0, "batch must be positive");
    require(y_dev && bits_dev, "null output pointer");
    SlotGenHost host;
    slotgen_prepare(*link, &host);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int L = link->n_taps, nch = link->has_interferer ? 2 : 1;
    const size_t tf = static_cast<size_t>(link->T) * link->F;
    // small per-call device scratch: pilots, tap profile, Jakes taps
    const size_t taps_bytes = static_cast<size_t>(B) * nch * link->T * link->N * L * sizeof(float2);
    const size_t bytes = tf + tf * sizeof(float2) + L * sizeof(float) + L * sizeof(double) + taps_bytes + 64;
    char* scratch = nullptr;
    CNRX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), bytes + 256, s));
    char* q = scratch;
    auto take = [&](size_t n) {
      char* r = q;
      q += (n + 15) & ~size_t(15);
      return r;
    };
    uint8_t* pmask = reinterpret_cast<uint8_t*>(take(tf));
    float2* pvals = reinterpret_cast<float2*>(take(tf * sizeof(float2)));
    float* gain = reinterpret_cast<float*>(take(L * sizeof(float)));
    double* tau = reinterpret_cast<double*>(take(L * sizeof(double)));
    float2* taps = reinterpret_cast<float2*>(take(taps_bytes));
    CNRX_CUDA(cudaMemcpyAsync(pmask, host.pmask.data(), tf, cudaMemcpyHostToDevice, s));
    CNRX_CUDA(cudaMemcpyAsync(pvals, host.pvals.data(), tf * sizeof(float2), cudaMemcpyHostToDevice, s));
    CNRX_CUDA(cudaMemcpyAsync(gain, host.gain.data(), L * sizeof(float), cudaMemcpyHostToDevice, s));
    CNRX_CUDA(cudaMemcpyAsync(tau, host.tau.data(), L * sizeof(double), cudaMemcpyHostToDevice, s));
    SlotGenArgs a{};
    a.B = B;
    a.T = link->T;
    a.F = link->F;
    a.N = link->N;
    a.L = L;
    a.nb = host.nb;
    a.has_interferer = link->has_interferer ? 1 : 0;
    a.scs = link->scs_hz;
    a.tsym = (1.0 + link->cp_fraction) / link->scs_hz;
    a.doppler_max = link->doppler_max_hz;
    a.snr_lo = link->snr_db_lo;
    a.snr_hi = link->snr_db_hi;
    a.sir_lo = link->sir_db_lo;
    a.sir_hi = link->sir_db_hi;
    a.seed = seed;
    a.slot0 = slot0;
    a.pmask = pmask;
    a.pvals = pvals;
    a.tap_gain = gain;
    a.tau = tau;
    slotgen_launch(a, taps, reinterpret_cast<float2*>(y_dev), bits_dev, reinterpret_cast<float2*>(h_dev), s);
    CNRX_CUDA(cudaFreeAsync(scratch, s));
    // host vectors of `host` are pageable: the copies above completed before cudaMemcpyAsync returned
  });
}

int cnrx_count_bit_errors(const float* llr_dev, const uint8_t* bits_dev, const uint8_t* data_mask_dev, int64_t B,
                          int64_t T, int64_t F, int32_t bits, unsigned long long* errors_dev, void* stream) {
  return guarded([&] {
    require(llr_dev && bits_dev && data_mask_dev && errors_dev, "null pointer");
    require(B > 0 && T > 0 && F > 0 && bits > 0, "dimensions must be positive");
    ber_launch(llr_dev, bits_dev, data_mask_dev, B, T * F * bits, bits, errors_dev, static_cast<cudaStream_t>(stream));
  });
}

int cnrx_slot_noise_var(const cnrx_link* link, int64_t B, uint64_t seed, uint64_t slot0, float* noise_var) {
  return guarded([&] {
    require(link != nullptr && noise_var != nullptr, "null pointer");
    require(B > 0, "batch must be positive");
    slot_noise_var(*link, B, seed, slot0, noise_var);
  });
}

int cnrx_classical_receive(cnrx_plan* plan, const float* y_dev, const float* h_dev, const float* noise_var_dev,
                           int64_t B, int64_t T, int64_t F, int64_t N, int32_t mod_order, float* llr_dev,
                           void* stream) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    require(y_dev && noise_var_dev && llr_dev, "null tensor pointer");
    require(B > 0 && T > 0 && F > 0 && N >= 1 && N <= 8, "bad grid dimensions");
    require(mod_order == 4 || mod_order == 16 || mod_order == 64, "modulation order must be 4, 16 or 64");
    const int bits = mod_order == 4 ? 2 : mod_order == 16 ? 4 : 6;
    DeviceGuard dg(plan->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : plan->stream;
    const float* feat = nullptr;
    if (!h_dev) {
      require(plan->has_pilots, "cnrx_set_pilots must be called before the LS-LMMSE receiver");
      require(T == plan->pT && F == plan->pF, "received grid does not match the pilot grid");
      // its own scratch (not the receive path's feat_buf, which a captured fp32 forward graph may point
      // at), ordered after the previous classical call when that ran on another stream
      const size_t bytes = static_cast<size_t>(B * T * F * 6 * N) * sizeof(float);
      if (plan->ws.classic_bytes < bytes && plan->classic_used) CNRX_CUDA(cudaEventSynchronize(plan->classic_done));
      float* f = static_cast<float*>(ensure_dev(plan->ws, plan->ws.classic_buf, plan->ws.classic_bytes, bytes));
      if (plan->classic_used && plan->classic_stream != s) CNRX_CUDA(cudaStreamWaitEvent(s, plan->classic_done, 0));
      PlaneGeom g = make_geom(static_cast<int>(B), static_cast<int>(T), static_cast<int>(F), 1);
      launch_featurize_ref(y_dev, g, static_cast<int>(N), plan->pt, f, s);
      feat = f;
    }
    launch_lmmse_demap(feat, reinterpret_cast<const float2*>(y_dev), reinterpret_cast<const float2*>(h_dev),
                       noise_var_dev, B, static_cast<int>(T), static_cast<int>(F), static_cast<int>(N), bits, llr_dev,
                       s);
    if (!h_dev) {
      if (!plan->classic_done) CNRX_CUDA(cudaEventCreateWithFlags(&plan->classic_done, cudaEventDisableTiming));
      CNRX_CUDA(cudaEventRecord(plan->classic_done, s));
      plan->classic_stream = s;
      plan->classic_used = true;
    }
  });
}

int cnrx_get_plan_info(const cnrx_plan* plan, cnrx_plan_info* info) {
  if (!plan || !info) return fail(CNRX_ERR_INVALID_ARGUMENT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->precision = plan->precision;
  info->device = plan->device;
  info->n_launches = static_cast<int32_t>(plan->launch_names.size());
  info->n_tc_convs = static_cast<int32_t>(plan->tc.size());
  info->input_channels = plan->in_ch;
  info->output_channels = plan->out_ch;
  info->macs_per_re = plan->macs;
  info->rows_per_slot = plan->ws.geo.P;
  size_t ws = 0;
  if (plan->precision != CNRX_FP32) {
    for (int c : plan->buf_channels) ws += static_cast<size_t>(plan->ws.geo.Nalloc) * c * 2;
  } else {
    for (int c : plan->f32_buf_channels) ws += static_cast<size_t>(plan->ws.B) * plan->ws.T * plan->ws.F * c * 4;
  }
  info->workspace_bytes = static_cast<int64_t>(ws);
  return CNRX_OK;
}

int cnrx_set_graph_capture(cnrx_plan* plan, int32_t enable) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> lk(plan->mu);
  plan->capture = enable != 0;
  if (!plan->capture && plan->gexec) {
    cudaGraphExecDestroy(plan->gexec);
    plan->gexec = nullptr;
    plan->gkey.clear();
  }
  return CNRX_OK;
}

int cnrx_set_profiling(cnrx_plan* plan, int32_t enable) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  std::lock_guard<std::mutex> lk(plan->mu);
  plan->profile = enable != 0;
  return CNRX_OK;
}

int cnrx_read_profile(cnrx_plan* plan, int32_t max_n, float* ms, int32_t* counts, int32_t* n_out) {
  if (!plan) return fail(CNRX_ERR_INVALID_ARGUMENT, "null plan");
  return guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    DeviceGuard dg(plan->device);
    for (auto& evs : plan->prof_events) {
      if (evs.empty()) continue;
      CNRX_CUDA(cudaEventSynchronize(evs.back()));
      for (size_t k = 1; k < evs.size(); ++k) {
        float t = 0.f;
        CNRX_CUDA(cudaEventElapsedTime(&t, evs[k - 1], evs[k]));
        if (plan->prof_ms.size() < k) {
          plan->prof_ms.resize(k, 0.0);
          plan->prof_count.resize(k, 0);
        }
        plan->prof_ms[k - 1] += t;
        plan->prof_count[k - 1] += 1;
      }
      for (auto e : evs) plan->event_pool.push_back(e);
    }
    plan->prof_events.clear();
    const int n = static_cast<int>(plan->prof_ms.size());
    if (n_out) *n_out = n;
    for (int i = 0; i < n && i < max_n; ++i) {
      if (ms) ms[i] = static_cast<float>(plan->prof_ms[static_cast<size_t>(i)]);
      if (counts) counts[i] = plan->prof_count[static_cast<size_t>(i)];
    }
    plan->prof_ms.clear();
    plan->prof_count.clear();
  });
}

int64_t cnrx_launch_flops(const cnrx_plan* plan, int32_t i) {
  if (!plan || i < 0 || i >= static_cast<int32_t>(plan->launch_flops.size())) return -1;
  return plan->launch_flops[static_cast<size_t>(i)];
}

const char* cnrx_launch_name(const cnrx_plan* plan, int32_t i) {
  if (!plan || i < 0 || i >= static_cast<int32_t>(plan->launch_names.size())) return nullptr;
  return plan->launch_names[static_cast<size_t>(i)].c_str();
}

int cnrx_ipc_alloc(int32_t device, int64_t bytes, void** ptr_out, cnrx_ipc_handle* handle_out) {
  if (!ptr_out || !handle_out || bytes <= 0) return fail(CNRX_ERR_INVALID_ARGUMENT, "bad argument");
  return guarded([&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(cnrx_ipc_handle), "CUDA IPC handle size");
    DeviceGuard dg(device);
    void* p = nullptr;
    CNRX_CUDA(cudaMalloc(&p, static_cast<size_t>(bytes)));  // its own allocation: the handle maps it from offset 0
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      throw Error(CNRX_ERR_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    }
    std::memcpy(handle_out->bytes, &h, sizeof h);
    *ptr_out = p;
  });
}

int cnrx_ipc_open(int32_t device, const cnrx_ipc_handle* handle, void** ptr_out) {
  if (!handle || !ptr_out) return fail(CNRX_ERR_INVALID_ARGUMENT, "null argument");
  return guarded([&] {
    DeviceGuard dg(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle->bytes, sizeof h);
    void* p = nullptr;
    CNRX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr_out = p;
  });
}

int cnrx_ipc_close(int32_t device, void* opened_ptr) {
  return guarded([&] {
    DeviceGuard dg(device);
    CNRX_CUDA(cudaIpcCloseMemHandle(opened_ptr));
  });
}

int cnrx_ipc_read(int32_t device, const void* src, void* host_dst, int64_t bytes) {
  if (!src || !host_dst || bytes < 0) return fail(CNRX_ERR_INVALID_ARGUMENT, "bad argument");
  return guarded([&] {
    DeviceGuard dg(device);
    CNRX_CUDA(cudaMemcpy(host_dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost));
  });
}

int cnrx_ipc_read_async(int32_t device, const void* src, void* host_dst, int64_t bytes, void* stream) {
  if (!src || !host_dst || bytes < 0) return fail(CNRX_ERR_INVALID_ARGUMENT, "bad argument");
  return guarded([&] {
    DeviceGuard dg(device);
    CNRX_CUDA(cudaMemcpyAsync(host_dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost,
                              static_cast<cudaStream_t>(stream)));
  });
}

int cnrx_ipc_free(int32_t device, void* allocated_ptr) {
  return guarded([&] {
    DeviceGuard dg(device);
    CNRX_CUDA(cudaFree(allocated_ptr));
  });
}

}  // extern "C"
