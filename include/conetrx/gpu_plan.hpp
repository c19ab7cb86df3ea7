// gpu_plan.hpp — C++ drop-in for conetrx::Network<float>::forward on B200 (header-only wrapper over
// the C ABI in conetrx_cuda.h).  Include it after the reference's "conetrx/network.hpp":
//
//     conetrx::Network<float> net = conetrx::build_conet<float>(spec);   // reference builder
//     ... load_checkpoint(net, path) / init_params / seed_norm_stats ...
//     conetrx::GpuPlan gpu(net, conetrx::GpuPlan::Precision::bf16, /*device=*/0);
//     Tensor<float> llr = gpu.forward(x, NormMode::eval);            // == net.forward(x, eval)
//
// What it mirrors (reference file:line):
//   * Network<T>::forward(const Tensor<T>&, NormMode, ...)  network.hpp:162-180 -> GpuPlan::forward
//   * GraphNode / nodes()                                     network.hpp:19-26, :335
//   * NamedParam / params()                                   network.hpp:28-33, :140
//   * bn_ready()                                              network.hpp:337
//   * errors: std::invalid_argument from require()            tensor.hpp:13-15
//             std::runtime_error for eval BN without stats   norms.hpp:66-69
// The plan copies (and for bf16 folds/converts) the weights at construction; like the reference's
// own object it is not re-entrant (one forward at a time per plan).
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "conetrx/network.hpp"
#include "conetrx_cuda.h"

namespace conetrx {

class GpuPlan {
 public:
  // bf16x3 / fp16x3: split-precision tensor-core plans, LLRs within 1e-4 relative of the fp32 forward
  enum class Precision { fp32 = CNRX_FP32, bf16 = CNRX_BF16, fp16 = CNRX_FP16, bf16x3 = CNRX_BF16X3, fp16x3 = CNRX_FP16X3 };

  // output_node: the index the network's set_output() named; -1 = recover it (see below).
  GpuPlan(Network<float>& net, Precision precision, int device = 0, int output_node = -1) {
    const auto& nodes = net.nodes();
    std::vector<cnrx_node> cn(nodes.size());
    int input = -1;
    std::vector<int> used(nodes.size(), 0);
    for (size_t i = 0; i < nodes.size(); ++i) {
      const GraphNode& n = nodes[i];
      cn[i] = cnrx_node{static_cast<int32_t>(n.op), n.in0, n.in1, n.w, n.b, n.gamma, n.beta, n.rmean, n.rvar,
                        n.bn_flag, n.out_channels, /*dilation_f=*/1};
      if (n.op == LayerOp::input) input = static_cast<int>(i);
      if (n.in0 >= 0) used[static_cast<size_t>(n.in0)] = 1;
      if (n.in1 >= 0) used[static_cast<size_t>(n.in1)] = 1;
    }
    // Network keeps output_node_ private; set_output() is always given the last unconsumed node by the
    // reference builders (network.hpp:482, :560), so recover it that way unless the caller names it, and
    // check the result against the output width the network reports (output_channels(), network.hpp:333):
    // a raw-API graph whose set_output() names another node must pass output_node explicitly.
    int output = output_node;
    for (int i = static_cast<int>(nodes.size()) - 1; i >= 0 && output < 0; --i)
      if (!used[static_cast<size_t>(i)]) output = i;
    if (output < 0 || output >= static_cast<int>(nodes.size()))
      throw std::invalid_argument("GpuPlan: bad output node index");
    if (nodes[static_cast<size_t>(output)].out_channels != net.output_channels())
      throw std::invalid_argument("GpuPlan: node " + std::to_string(output) + " has " +
                                  std::to_string(nodes[static_cast<size_t>(output)].out_channels) +
                                  " channels but the network's output has " + std::to_string(net.output_channels()) +
                                  "; pass the set_output() node index explicitly");
    const auto& params = net.params();
    std::vector<cnrx_param> cp(params.size());
    for (size_t i = 0; i < params.size(); ++i) {
      const auto& p = params[i];
      cnrx_param q{};
      q.name = p.name.c_str();
      q.rank = p.value.rank();
      q.learnable = p.learnable ? 1 : 0;
      for (int d = 0; d < p.value.rank() && d < 4; ++d) q.dims[d] = p.value.dim(d);
      q.data = p.value.data();
      cp[i] = q;
    }
    const auto& ready = net.bn_ready();
    check(cnrx_plan_create(cn.data(), static_cast<int32_t>(cn.size()), input, output, cp.data(),
                           static_cast<int32_t>(cp.size()), ready.data(), static_cast<int32_t>(ready.size()),
                           static_cast<int32_t>(precision), device, &plan_));
    out_channels_ = nodes[static_cast<size_t>(output)].out_channels;
  }
  ~GpuPlan() { cnrx_plan_destroy(plan_); }
  GpuPlan(const GpuPlan&) = delete;
  GpuPlan& operator=(const GpuPlan&) = delete;

  // Network<float>::forward(x, mode) (network.hpp:162): x [B,T,F,C] or [T,F,C] channels-last.
  Tensor<float> forward(const Tensor<float>& x, NormMode mode) {
    ActDims d = act_dims(x);  // same shape check / message as the reference (kernels.hpp:17-21)
    std::vector<int64_t> shape = x.shape();
    shape.back() = out_channels_;
    Tensor<float> y(shape);
    check(cnrx_forward(plan_, x.data(), d.b, d.t, d.f, d.c, mode == NormMode::eval ? CNRX_MODE_EVAL : CNRX_MODE_TRAIN,
                       y.data()));
    return y;
  }

  // Receiver path: y [B,T,F,N] complex (interleaved re/im floats), pilots [T,F] complex + mask.
  void set_pilots(int64_t T, int64_t F, const float* pilots, const uint8_t* mask) {
    check(cnrx_set_pilots(plan_, T, F, pilots, mask));
  }
  void receive(const float* y, int64_t B, int64_t T, int64_t F, int64_t N, float* llr) {
    check(cnrx_receive(plan_, y, B, T, F, N, llr));
  }

  cnrx_plan* handle() { return plan_; }

 private:
  static void check(int rc) {
    if (rc == CNRX_OK) return;
    const std::string msg = cnrx_last_error();
    if (rc == CNRX_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);  // not-ready (norms.hpp:66-69), unsupported, CUDA errors
  }
  cnrx_plan* plan_ = nullptr;
  int out_channels_ = 0;
};

}  // namespace conetrx
