// drop_in_example.cpp — the reference-side integration, end to end in C++: build a CoNet-Rx network
// with the reference's OWN builders (conetrx::conet_template + build_conet), initialise it with the
// reference's Rng, run the reference CPU forward and the B200 plan through include/conetrx/gpu_plan.hpp
// on the same input, and compare.  Built by tools/integration/Makefile into oracle/_ref/ (it compiles
// against the reference headers, so it is reference-side code, not part of the product).
#include <cmath>
#include <cstdio>

#include "conetrx/gpu_plan.hpp"
#include "conetrx/network.hpp"

int main() {
  using namespace conetrx;
  auto spec = conet_template(64, 4, {4, 4}, FusionOp::mul, NormKind::batch, false, 12, 4, ConvKind::standard, 3,
                             {3});
  spec.main.kernel = 1;
  for (auto& s : spec.supports) s.kernel = 1;
  Network<float> net = build_conet<float>(spec);
  Rng rng(2024);
  net.init_params(rng);
  net.seed_norm_stats();

  const int64_t B = 2, T = 14, F = 64, C = 12;
  Tensor<float> x({B, T, F, C});
  Rng xr(7);
  for (auto& v : x.vec()) v = static_cast<float>(xr.normal());

  Tensor<float> ref = net.forward(x, NormMode::eval);
  int rc = 0;
  for (auto prec : {GpuPlan::Precision::fp32, GpuPlan::Precision::bf16}) {
    GpuPlan gpu(net, prec, 0);
    Tensor<float> y = gpu.forward(x, NormMode::eval);
    double num = 0, den = 0, maxabs = 0;
    size_t agree = 0;
    for (int64_t i = 0; i < y.numel(); ++i) {
      const double d = static_cast<double>(y[i]) - ref[i];
      num += d * d;
      den += static_cast<double>(ref[i]) * ref[i];
      maxabs = std::max(maxabs, std::fabs(d));
      agree += (y[i] > 0) == (ref[i] > 0);
    }
    const double rel = std::sqrt(num / den);
    const double frac = static_cast<double>(agree) / static_cast<double>(y.numel());
    std::printf("%s: rel L2 %.3e  max abs %.3e  sign agreement %.5f\n",
                prec == GpuPlan::Precision::fp32 ? "fp32" : "bf16", rel, maxabs, frac);
    if (prec == GpuPlan::Precision::fp32 && maxabs != 0.0) rc = 1;  // fp32 plan is bit-exact
    if (prec == GpuPlan::Precision::bf16 && (rel > 3e-2 || frac < 0.99)) rc = 1;
  }
  // error semantics: wrong channel count -> std::invalid_argument, like Network::forward
  try {
    GpuPlan gpu(net, GpuPlan::Precision::bf16, 0);
    Tensor<float> bad({1, T, F, 10});
    gpu.forward(bad, NormMode::eval);
    rc = 1;
  } catch (const std::invalid_argument& e) {
    std::printf("invalid_argument as expected: %s\n", e.what());
  }
  std::printf(rc == 0 ? "drop-in OK\n" : "drop-in FAILED\n");
  return rc;
}
