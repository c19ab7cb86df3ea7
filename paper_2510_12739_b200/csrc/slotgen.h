// slotgen.h — on-GPU synthetic slots + bit-error counting (slotgen.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../../include/conetrx_cuda.h"

namespace cnrx {

// Host-side preparation shared by every launch of one link: pilot grid, tap gains / delays.
struct SlotGenHost {
  int nb = 0;
  std::vector<uint8_t> pmask;  // [T*F]
  std::vector<float> pvals;    // [T*F][2]
  std::vector<float> gain;     // [L] sqrt(p_l / 20)
  std::vector<double> tau;     // [L] seconds
};

struct SlotGenArgs {
  int64_t B;
  int T, F, N, L, nb, has_interferer;
  double scs, tsym, doppler_max, snr_lo, snr_hi, sir_lo, sir_hi;
  uint64_t seed, slot0;
  const uint8_t* pmask;  // device [T*F]
  const float2* pvals;   // device [T*F]
  const float* tap_gain; // device [L]
  const double* tau;     // device [L]
};

void slotgen_prepare(const cnrx_link& link, SlotGenHost* h);
// host restatement of the per-slot draws: total noise + interference variance of slots slot0 .. slot0+B-1
void slot_noise_var(const cnrx_link& link, int64_t B, uint64_t seed, uint64_t slot0, float* out);
// taps: device scratch of B * (1 + has_interferer) * T * N * L float2
void slotgen_launch(const SlotGenArgs& a, float2* taps, float2* y, uint8_t* bits, float2* h, cudaStream_t s);
void ber_launch(const float* llr, const uint8_t* bits, const uint8_t* data_mask, int64_t B, int64_t per_slot, int nb,
                unsigned long long* errors, cudaStream_t s);

}  // namespace cnrx
