// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the oracle). Never linked into the product.
//
// A C-ABI shim around the UNMODIFIED reference C++ library (proj/core of arxiv/paper_2510_12739),
// compiled in place from /root/reference by oracle/Makefile into oracle/_ref/libconetrx_ref.so.
// It exposes exactly the reference objects the CoNet-Rx inference path uses:
//   * conetrx::Network<float> construction (network.hpp:49-112), builders build_conet / build_net
//     (network.hpp:470-562) and the templates (netspec.cpp:42-81);
//   * Network<float>::forward / forward_concurrent (network.hpp:162-212) — the hot path we replace;
//   * the host-side PHY helpers used to pin the synthetic-slot generator: Rng (rng.hpp:14-69),
//     qam_map (qam.cpp:42-52), pilot_pattern (pilots.cpp:13-31), tdl_channel (channel.cpp:52-111);
//   * param_count / solve_filters (netspec.cpp:99-153) and CNCK checkpoints (checkpoint.cpp:47-99).
// Every call catches the reference's exceptions and maps them to status codes + a message so the
// Python tests can assert the reference's own error behaviour.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "conetrx/channel.hpp"
#include "conetrx/netspec.hpp"
#include "conetrx/network.hpp"
#include "conetrx/pilots.hpp"
#include "conetrx/qam.hpp"
#include "conetrx/rng.hpp"

using conetrx::Network;
using conetrx::Tensor;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Network<float>* net(void* h) { return static_cast<Network<float>*>(h); }
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------------------------------------
// Network construction (network.hpp:49-112). All return a node index, or -1 with ref_last_error().
// ---------------------------------------------------------------------------------------------
void* ref_net_new() { return new Network<float>(); }
void ref_net_free(void* h) { delete net(h); }

int ref_add_input(void* h, int ch) {
  int r = -1;
  if (guarded([&] { r = net(h)->add_input(ch); })) return -1;
  return r;
}
int ref_add_conv(void* h, int in, const char* name, int kernel, int cin, int cout, int bias) {
  int r = -1;
  if (guarded([&] { r = net(h)->add_conv(in, name, kernel, cin, cout, bias != 0); })) return -1;
  return r;
}
int ref_add_dwconv(void* h, int in, const char* name, int kernel, int c, int bias) {
  int r = -1;
  if (guarded([&] { r = net(h)->add_dwconv(in, name, kernel, c, bias != 0); })) return -1;
  return r;
}
int ref_add_relu(void* h, int in) {
  int r = -1;
  if (guarded([&] { r = net(h)->add_relu(in); })) return -1;
  return r;
}
int ref_add_norm(void* h, int in, int kind, const char* name, int ch) {
  int r = -1;
  if (guarded([&] {
        r = net(h)->add_norm(in, kind == 0 ? conetrx::NormKind::batch : conetrx::NormKind::layer, name, ch);
      }))
    return -1;
  return r;
}
// op: 6 = add, 7 = mul (LayerOp values)
int ref_add_binary(void* h, int op, int a, int b) {
  int r = -1;
  if (guarded([&] {
        r = net(h)->add_binary(op == 7 ? conetrx::LayerOp::mul : conetrx::LayerOp::add, a, b);
      }))
    return -1;
  return r;
}
int ref_add_concat(void* h, int a, int b) {
  int r = -1;
  if (guarded([&] { r = net(h)->add_concat(a, b); })) return -1;
  return r;
}
void ref_set_output(void* h, int node) { net(h)->set_output(node); }

// conet_template (netspec.cpp:53-81) + build_conet (network.hpp:490-562).
// fusion_op 0 mul / 1 add / 2 concat; norm 0 bn / 1 ln; conv_kind 0 standard / 1 depthwise.
void* ref_build_conet(int width, int main_blocks, const int* support_blocks, int n_sup, int fusion_op, int norm,
                      int bidir, int in_ch, int bits, int conv_kind, int kernel, const int* fusion_points,
                      int n_fp) {
  Network<float>* out = nullptr;
  int rc = guarded([&] {
    std::vector<int> sb(support_blocks, support_blocks + n_sup);
    std::vector<int> fp(fusion_points, fusion_points + n_fp);
    auto spec = conetrx::conet_template(
        width, main_blocks, sb, static_cast<conetrx::FusionOp>(fusion_op), static_cast<conetrx::NormKind>(norm),
        bidir != 0, in_ch, bits, static_cast<conetrx::ConvKind>(conv_kind), kernel, fp);
    out = new Network<float>(conetrx::build_conet<float>(spec));
  });
  return rc ? nullptr : out;
}

// Same, but the spec's NetSpec.kernel (stem/head) and BlockSpec.kernel (blocks) set independently —
// the BASELINE configs use 1x1 stems/heads with 3x3 blocks.
void* ref_build_conet_k(int width, int main_blocks, const int* support_blocks, int n_sup, int fusion_op, int norm,
                        int bidir, int in_ch, int bits, int block_kind, int io_kernel, int block_kernel,
                        const int* fusion_points, int n_fp) {
  Network<float>* out = nullptr;
  int rc = guarded([&] {
    std::vector<int> sb(support_blocks, support_blocks + n_sup);
    std::vector<int> fp(fusion_points, fusion_points + n_fp);
    auto spec = conetrx::conet_template(width, main_blocks, sb, static_cast<conetrx::FusionOp>(fusion_op),
                                        static_cast<conetrx::NormKind>(norm), bidir != 0, in_ch, bits,
                                        conetrx::ConvKind::standard, block_kernel, fp);
    spec.main.kernel = io_kernel;
    for (auto& b : spec.main.blocks) b.kind = static_cast<conetrx::BlockKind>(block_kind);
    for (auto& s : spec.supports) {
      s.kernel = io_kernel;
      for (auto& b : s.blocks) b.kind = static_cast<conetrx::BlockKind>(block_kind);
    }
    out = new Network<float>(conetrx::build_conet<float>(spec));
  });
  return rc ? nullptr : out;
}

// deeprx_template (netspec.cpp:42-51) + build_net (network.hpp:470-483), with separate io/block kernels.
void* ref_build_deeprx_k(int width, int blocks, int in_ch, int bits, int block_kind, int io_kernel,
                         int block_kernel) {
  Network<float>* out = nullptr;
  int rc = guarded([&] {
    auto spec = conetrx::deeprx_template(width, blocks, in_ch, bits, conetrx::ConvKind::standard, block_kernel);
    spec.kernel = io_kernel;
    for (auto& b : spec.blocks) b.kind = static_cast<conetrx::BlockKind>(block_kind);
    out = new Network<float>(conetrx::build_net<float>(spec));
  });
  return rc ? nullptr : out;
}

// ---------------------------------------------------------------------------------------------
// Introspection (GraphNode network.hpp:19-26; NamedParam :28-33)
// ---------------------------------------------------------------------------------------------
int ref_n_nodes(void* h) { return net(h)->n_nodes(); }
// out[11] = op,in0,in1,w,b,gamma,beta,rmean,rvar,bn_flag,out_channels
void ref_get_node(void* h, int i, int* o) {
  const auto& n = net(h)->nodes()[static_cast<size_t>(i)];
  int v[11] = {static_cast<int>(n.op), n.in0, n.in1, n.w, n.b, n.gamma, n.beta, n.rmean, n.rvar, n.bn_flag,
               n.out_channels};
  std::memcpy(o, v, sizeof(v));
}
int ref_output_node(void* h) {
  // output node = the node whose out_channels equal output_channels and that nothing consumes (last set_output).
  // The reference keeps output_node_ private; recover it as the last node with no consumer.
  const auto& nodes = net(h)->nodes();
  std::vector<int> used(nodes.size(), 0);
  for (const auto& n : nodes) {
    if (n.in0 >= 0) used[static_cast<size_t>(n.in0)] = 1;
    if (n.in1 >= 0) used[static_cast<size_t>(n.in1)] = 1;
  }
  for (int i = static_cast<int>(nodes.size()) - 1; i >= 0; --i)
    if (!used[static_cast<size_t>(i)]) return i;
  return -1;
}
int ref_n_params(void* h) { return static_cast<int>(net(h)->params().size()); }
const char* ref_param_name(void* h, int i) { return net(h)->params()[static_cast<size_t>(i)].name.c_str(); }
int ref_param_rank(void* h, int i) { return net(h)->params()[static_cast<size_t>(i)].value.rank(); }
int64_t ref_param_dim(void* h, int i, int d) { return net(h)->params()[static_cast<size_t>(i)].value.dim(d); }
int ref_param_learnable(void* h, int i) { return net(h)->params()[static_cast<size_t>(i)].learnable ? 1 : 0; }
float* ref_param_data(void* h, int i) { return net(h)->params()[static_cast<size_t>(i)].value.data(); }
int ref_n_bn(void* h) { return static_cast<int>(net(h)->bn_ready().size()); }
void ref_set_bn_ready(void* h, int i, int v) { net(h)->bn_ready()[static_cast<size_t>(i)] = static_cast<uint8_t>(v); }
int ref_get_bn_ready(void* h, int i) { return net(h)->bn_ready()[static_cast<size_t>(i)]; }
void ref_seed_norm_stats(void* h) { net(h)->seed_norm_stats(); }
int64_t ref_learnable_count(void* h) { return net(h)->learnable_count(); }
int ref_conv_depth(void* h) { return net(h)->conv_depth(); }
int ref_init_params(void* h, uint64_t seed) {
  return guarded([&] {
    conetrx::Rng rng(seed);
    net(h)->init_params(rng);
  });
}

// ---------------------------------------------------------------------------------------------
// The hot path: Network<float>::forward (network.hpp:162) / forward_concurrent (:186).
// x is [B,T,F,C] fp32 (tensor.hpp:17-19); out must hold B*T*F*output_channels floats.
// mode 0 = eval, 1 = train. Returns 0, or 1 invalid_argument / 2 runtime_error.
// ---------------------------------------------------------------------------------------------
int ref_forward(void* h, const float* x, int64_t B, int64_t T, int64_t F, int64_t C, float* out, int concurrent,
                int mode) {
  return guarded([&] {
    Tensor<float> xt({B, T, F, C}, std::vector<float>(x, x + B * T * F * C));
    const auto m = mode == 1 ? conetrx::NormMode::train : conetrx::NormMode::eval;
    Tensor<float> y = concurrent ? net(h)->forward_concurrent(xt, m) : net(h)->forward(xt, m);
    std::memcpy(out, y.data(), static_cast<size_t>(y.numel()) * sizeof(float));
  });
}

// Forward with node overrides (network.hpp:159-178): node ids + fill values (fusion-identity tests).
int ref_forward_overrides(void* h, const float* x, int64_t B, int64_t T, int64_t F, int64_t C, float* out,
                          const int* ids, const float* vals, int n) {
  return guarded([&] {
    Tensor<float> xt({B, T, F, C}, std::vector<float>(x, x + B * T * F * C));
    std::map<int, float> ov;
    for (int i = 0; i < n; ++i) ov[ids[i]] = vals[i];
    Tensor<float> y = net(h)->forward(xt, conetrx::NormMode::eval, nullptr, &ov);
    std::memcpy(out, y.data(), static_cast<size_t>(y.numel()) * sizeof(float));
  });
}

// Wall-clock of `reps` forward calls (steady_clock, seconds), for the CPU baseline leg.
double ref_time_forward(void* h, const float* x, int64_t B, int64_t T, int64_t F, int64_t C, float* out,
                        int concurrent, int reps) {
  Tensor<float> xt({B, T, F, C}, std::vector<float>(x, x + B * T * F * C));
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) {
    Tensor<float> y = concurrent ? net(h)->forward_concurrent(xt, conetrx::NormMode::eval)
                                 : net(h)->forward(xt, conetrx::NormMode::eval);
    if (r == reps - 1) std::memcpy(out, y.data(), static_cast<size_t>(y.numel()) * sizeof(float));
  }
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

int ref_threads() { return conetrx::Compute::effective_threads(); }

// ---------------------------------------------------------------------------------------------
// Checkpoints (checkpoint.cpp:47-99)
// ---------------------------------------------------------------------------------------------
int ref_save_checkpoint(void* h, const char* path) {
  return guarded([&] { conetrx::save_checkpoint(*net(h), path); });
}
int ref_load_checkpoint(void* h, const char* path) {
  return guarded([&] { conetrx::load_checkpoint(*net(h), path); });
}


// ---------------------------------------------------------------------------------------------
// Spec files (netspec.cpp:160-257): JSON -> SpecFile -> canonical JSON / network / width solve
// ---------------------------------------------------------------------------------------------
int ref_spec_to_json(const char* text, char* out, int cap) {
  return guarded([&] {
    const std::string j = conetrx::spec_file_to_json(conetrx::parse_spec_file_json(text));
    if (static_cast<int>(j.size()) + 1 > cap) throw std::runtime_error("output buffer too small");
    std::memcpy(out, j.c_str(), j.size() + 1);
  });
}
void* ref_net_from_spec(const char* text) {
  Network<float>* out = nullptr;
  int rc = guarded([&] {
    const conetrx::SpecFile f = conetrx::parse_spec_file_json(text);
    out = f.is_conet() ? new Network<float>(conetrx::build_conet<float>(f.to_conet()))
                       : new Network<float>(conetrx::build_net<float>(f.to_deeprx()));
  });
  return rc ? nullptr : out;
}
int ref_solve_spec_width(const char* text, long long target, double tol, int* found, int* width,
                         long long* params, int* lo_w, int* hi_w) {
  return guarded([&] {
    const auto r = conetrx::solve_spec_width(conetrx::parse_spec_file_json(text), target, tol);
    *found = r.found ? 1 : 0;
    *width = r.width;
    *params = r.params;
    *lo_w = r.lo_width;
    *hi_w = r.hi_width;
  });
}

// ---------------------------------------------------------------------------------------------
// PHY helpers used to pin the synthetic-slot generator restatement
// ---------------------------------------------------------------------------------------------
void ref_rng_u64(uint64_t seed, int n, uint64_t* out) {
  conetrx::Rng rng(seed);
  for (int i = 0; i < n; ++i) out[i] = rng.next_u64();
}
void ref_rng_uniform(uint64_t seed, int n, double* out) {
  conetrx::Rng rng(seed);
  for (int i = 0; i < n; ++i) out[i] = rng.uniform();
}
void ref_rng_normal(uint64_t seed, int n, double* out) {
  conetrx::Rng rng(seed);
  for (int i = 0; i < n; ++i) out[i] = rng.normal();
}
uint64_t ref_rng_derive(uint64_t master, uint64_t index) { return conetrx::Rng::derive(master, index); }

int ref_qam_map(const uint8_t* bits, int order, double* re_im) {
  return guarded([&] {
    auto s = conetrx::qam_map(bits, order);
    re_im[0] = s.real();
    re_im[1] = s.imag();
  });
}

// pilot_pattern for a LinkConfig with T, F and PilotConfig{symbol_index, spacing}. values re/im [T*F*2].
int ref_pilot_pattern(int T, int F, int symbol_index, int spacing, uint8_t* mask, double* values) {
  return guarded([&] {
    conetrx::LinkConfig cfg;
    cfg.T = T;
    cfg.F = F;
    cfg.pilot.symbol_index = symbol_index;
    cfg.pilot.spacing = spacing;
    auto p = conetrx::pilot_pattern(cfg);
    for (int i = 0; i < T * F; ++i) {
      mask[i] = p.mask[static_cast<size_t>(i)];
      values[2 * i] = p.values[static_cast<size_t>(i)].real();
      values[2 * i + 1] = p.values[static_cast<size_t>(i)].imag();
    }
  });
}

// tdl_channel with the reference's fixed 16 taps on the 1/(F*df) grid. grid re/im [T*F*N*2].
int ref_tdl_channel(double delay_spread_s, double speed_mps, int T, int F, int N, double scs_hz, double fc_hz,
                    double cp_fraction, uint64_t seed, double* grid, double* tap_powers, double* doppler_hz) {
  return guarded([&] {
    conetrx::LinkConfig cfg;
    cfg.T = T;
    cfg.F = F;
    cfg.N = N;
    cfg.subcarrier_spacing_hz = scs_hz;
    cfg.carrier_freq_hz = fc_hz;
    cfg.cp_fraction = cp_fraction;
    conetrx::Rng rng(seed);
    auto link = conetrx::tdl_channel(delay_spread_s, speed_mps, cfg, rng);
    for (size_t i = 0; i < link.grid.size(); ++i) {
      grid[2 * i] = link.grid[i].real();
      grid[2 * i + 1] = link.grid[i].imag();
    }
    for (size_t l = 0; l < link.tap_powers.size(); ++l) tap_powers[l] = link.tap_powers[l];
    *doppler_hz = link.doppler_hz;
  });
}

void ref_tdl_tap_powers(double delay_spread_s, double spacing_s, int n_taps, double* out) {
  auto p = conetrx::tdl_tap_powers(delay_spread_s, spacing_s, n_taps);
  for (int i = 0; i < n_taps; ++i) out[i] = p[static_cast<size_t>(i)];
}

// param_count of the conet template (netspec.cpp:99-101), total + sequential depth.
int ref_param_count_conet(int width, int main_blocks, const int* support_blocks, int n_sup, int in_ch, int bits,
                          int kernel, int64_t* total, int* depth) {
  return guarded([&] {
    std::vector<int> sb(support_blocks, support_blocks + n_sup);
    auto spec = conetrx::conet_template(width, main_blocks, sb, conetrx::FusionOp::mul, conetrx::NormKind::batch,
                                        false, in_ch, bits, conetrx::ConvKind::standard, kernel, {});
    auto rep = conetrx::param_count(spec);
    *total = rep.total_learnable;
    *depth = rep.sequential_conv_depth;
  });
}

}  // extern "C"
