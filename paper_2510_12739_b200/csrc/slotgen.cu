// slotgen.cu — on-GPU synthetic OFDM slots and bit-error counting.
//
// The reference's slot model (SPEC.md:212-220 generate_tti; Gray QAM qam.cpp:10-52; pilots
// pilots.cpp:13-31 on the DM-RS symbols; TDL channel with an exponential PDP and per-tap Jakes
// processes channel.cpp:37-111; AWGN at a per-slot SNR; a co-channel QPSK interferer for config 3)
// generated where the receiver runs, so BER sweeps and throughput runs never cross PCIe.  Every random
// draw is a Philox4x32-10 block addressed by (index, purpose, slot) under the run's seed, so slots and
// resource elements are generated independently in parallel and any slot can be regenerated alone.
// The CPU restatement (test infrastructure) is oracle/slotgen.py; the layout of the draws is documented
// there.
//
// Kernels: (1) per (slot, channel, symbol, antenna, tap) the Jakes sum of 20 sinusoids; (2) per
// (slot, symbol, subcarrier) bits, QAM / pilot symbol, H = sum_l a_l(t) e^{-j 2 pi f df tau_l} per
// antenna, interferer, noise -> y; (3) per-slot hard-decision error counts over data REs.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "common.h"
#include "slotgen.h"

namespace cnrx {

namespace {

constexpr int kSin = 20;
enum : uint32_t { P_SLOT = 1, P_BITS = 2, P_JAKES = 3, P_JAKES_I = 4, P_NOISE = 5, P_IBITS = 6 };

struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = 0xD2511F53ull * c0, p1 = 0xCD9E8D57ull * c2;
    const uint32_t lo0 = static_cast<uint32_t>(p0), hi0 = static_cast<uint32_t>(p0 >> 32);
    const uint32_t lo1 = static_cast<uint32_t>(p1), hi1 = static_cast<uint32_t>(p1 >> 32);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return U4{c0, c1, c2, c3};
}

struct Draw {
  uint32_t k0, k1, s0, s1;
  __device__ U4 operator()(uint32_t purpose, uint32_t index) const { return philox(index, purpose, s0, s1, k0, k1); }
};

__host__ __device__ __forceinline__ float unif(uint32_t w) { return static_cast<float>(w >> 8) * 5.9604644775390625e-8f; }

__device__ __forceinline__ Draw draw_for(const SlotGenArgs& a, int64_t b) {
  const uint64_t slot = a.slot0 + static_cast<uint64_t>(b);
  return Draw{static_cast<uint32_t>(a.seed), static_cast<uint32_t>(a.seed >> 32), static_cast<uint32_t>(slot),
              static_cast<uint32_t>(slot >> 32)};
}

// QAM axis level from the bits of one axis (qam.cpp:23-30), unnormalised
__device__ __forceinline__ float axis_level(uint32_t v0, uint32_t v1, uint32_t v2, int half) {
  const float s0 = 1.f - 2.f * static_cast<float>(v0);
  if (half == 1) return s0;
  const float s1 = 1.f - 2.f * static_cast<float>(v1);
  if (half == 2) return s0 * (2.f - s1);
  const float s2 = 1.f - 2.f * static_cast<float>(v2);
  return s0 * (4.f - s1 * (2.f - s2));
}

__device__ __forceinline__ float2 qam(uint32_t w, int nb) {
  const int half = nb / 2;
  const float i = axis_level(w & 1u, (w >> 2) & 1u, (w >> 4) & 1u, half);
  const float q = axis_level((w >> 1) & 1u, (w >> 3) & 1u, (w >> 5) & 1u, half);
  const float nf = nb == 2 ? 0.70710678118654752f : nb == 4 ? 0.31622776601683794f : 0.15430334996209191f;
  return make_float2(i * nf, q * nf);
}

// taps[b][ch][t][n][l] = sqrt(p_l / S) sum_s exp(j (w_s t Tsym + phi_s))
__global__ void taps_kernel(const SlotGenArgs a, float2* taps) {
  const int nch = a.has_interferer ? 2 : 1;
  const int64_t total = a.B * nch * a.T * a.N * a.L;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = i;
    const int l = static_cast<int>(r % a.L);
    r /= a.L;
    const int n = static_cast<int>(r % a.N);
    r /= a.N;
    const int t = static_cast<int>(r % a.T);
    r /= a.T;
    const int ch = static_cast<int>(r % nch);
    const int64_t b = r / nch;
    const Draw d = draw_for(a, b);
    const U4 ws = d(P_SLOT, 0);
    const float fd = a.doppler_max > 0 ? static_cast<float>(a.doppler_max) * unif(ws.y) : 0.f;
    const float tt = static_cast<float>(t * a.tsym);
    float re = 0.f, im = 0.f;
    for (int s = 0; s < kSin; ++s) {
      const U4 w = d(ch == 0 ? P_JAKES : P_JAKES_I, static_cast<uint32_t>((n * a.L + l) * kSin + s));
      const float omega = 6.28318530717958648f * fd * cospif(2.f * unif(w.x));
      const float arg = omega * tt + 6.28318530717958648f * unif(w.y);
      float sn, cs;
      sincosf(arg, &sn, &cs);
      re += cs;
      im += sn;
    }
    const float g = a.tap_gain[l];
    taps[i] = make_float2(re * g, im * g);
  }
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }

// one thread per (slot, symbol, subcarrier)
__global__ void re_kernel(const SlotGenArgs a, const float2* __restrict__ taps, float2* __restrict__ y,
                          uint8_t* __restrict__ bits, float2* __restrict__ hout) {
  const int nch = a.has_interferer ? 2 : 1;
  const int64_t total = a.B * a.T * a.F;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int f = static_cast<int>(i % a.F);
    const int t = static_cast<int>((i / a.F) % a.T);
    const int64_t b = i / (static_cast<int64_t>(a.F) * a.T);
    const int re_idx = t * a.F + f;
    const Draw d = draw_for(a, b);
    const U4 ws = d(P_SLOT, 0);
    const float snr = static_cast<float>(a.snr_lo + (a.snr_hi - a.snr_lo) * static_cast<double>(unif(ws.x)));
    const float nsd = sqrtf(0.5f * exp10f(-snr / 10.f));
    float2 x;
    uint32_t wb = d(P_BITS, static_cast<uint32_t>(re_idx)).x & ((1u << a.nb) - 1u);
    if (a.pmask[re_idx]) {
      wb = 0;
      x = a.pvals[re_idx];
    } else {
      x = qam(wb, a.nb);
    }
    uint8_t* bo = bits + i * a.nb;
    for (int k = 0; k < a.nb; ++k) bo[k] = static_cast<uint8_t>((wb >> k) & 1u);
    float2 z = make_float2(0.f, 0.f);
    if (a.has_interferer) {
      const float sir = static_cast<float>(a.sir_lo + (a.sir_hi - a.sir_lo) * static_cast<double>(unif(ws.z)));
      z = qam(d(P_IBITS, static_cast<uint32_t>(re_idx)).x & 3u, 2);
      const float amp = sqrtf(exp10f(-sir / 10.f));
      z.x *= amp;
      z.y *= amp;
    }
    for (int n = 0; n < a.N; ++n) {
      float2 h = make_float2(0.f, 0.f), g = make_float2(0.f, 0.f);
      for (int l = 0; l < a.L; ++l) {
        double ph = static_cast<double>(f) * a.scs * a.tau[l];
        ph -= floor(ph);
        float sn, cs;
        sincospif(-2.f * static_cast<float>(ph), &sn, &cs);
        const float2 tw = make_float2(cs, sn);
        const float2 a0 = taps[(((b * nch + 0) * a.T + t) * a.N + n) * a.L + l];
        h = make_float2(h.x + a0.x * tw.x - a0.y * tw.y, h.y + a0.x * tw.y + a0.y * tw.x);
        if (a.has_interferer) {
          const float2 a1 = taps[(((b * nch + 1) * a.T + t) * a.N + n) * a.L + l];
          g = make_float2(g.x + a1.x * tw.x - a1.y * tw.y, g.y + a1.x * tw.y + a1.y * tw.x);
        }
      }
      float2 v = cmul(h, x);
      if (a.has_interferer) {
        const float2 gz = cmul(g, z);
        v.x += gz.x;
        v.y += gz.y;
      }
      const U4 wn = d(P_NOISE, static_cast<uint32_t>(re_idx * a.N + n));
      const float r = sqrtf(-2.f * logf((static_cast<float>(wn.x >> 8) + 1.f) * 5.9604644775390625e-8f));
      float sn, cs;
      sincospif(2.f * unif(wn.y), &sn, &cs);
      v.x += r * cs * nsd;
      v.y += r * sn * nsd;
      y[i * a.N + n] = v;
      if (hout) hout[i * a.N + n] = h;
    }
  }
}

// per-slot hard-decision errors over data REs: LLR > 0 => bit 1
__global__ void ber_kernel(const float* __restrict__ llr, const uint8_t* __restrict__ bits,
                           const uint8_t* __restrict__ data_mask, int64_t per_slot, int nb,
                           unsigned long long* __restrict__ errors) {
  const int64_t b = blockIdx.y;
  unsigned int cnt = 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < per_slot;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!data_mask[e / nb]) continue;
    const uint8_t hard = llr[b * per_slot + e] > 0.f ? 1 : 0;
    cnt += hard != bits[b * per_slot + e];
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ unsigned int part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x < 32) {
    unsigned int v = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0u;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0 && v) atomicAdd(&errors[b], static_cast<unsigned long long>(v));
  }
}

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// tdl_tap_powers (channel.cpp:37-50): exponential PDP, decay bisected in log space to the RMS spread
std::vector<double> tap_powers(double rms, double spacing, int n) {
  auto powers = [&](double beta) {
    std::vector<double> p(static_cast<size_t>(n));
    double s = 0;
    for (int l = 0; l < n; ++l) s += (p[static_cast<size_t>(l)] = std::exp(-l * spacing / beta));
    for (double& v : p) v /= s;
    return p;
  };
  auto spread = [&](const std::vector<double>& p) {
    double m1 = 0, m2 = 0;
    for (int l = 0; l < n; ++l) {
      const double tau = l * spacing;
      m1 += p[static_cast<size_t>(l)] * tau;
      m2 += p[static_cast<size_t>(l)] * tau * tau;
    }
    const double v = m2 - m1 * m1;
    return v > 0 ? std::sqrt(v) : 0.0;
  };
  double lo = std::log(1e-12), hi = 0.0;
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (spread(powers(std::exp(mid))) < rms) lo = mid;
    else hi = mid;
  }
  return powers(std::exp(0.5 * (lo + hi)));
}

}  // namespace

void slotgen_prepare(const cnrx_link& link, SlotGenHost* h) {
  require(link.T > 0 && link.F > 0 && link.N > 0 && link.n_taps > 0, "link dimensions must be positive");
  require(link.mod_order == 4 || link.mod_order == 16 || link.mod_order == 64, "modulation order must be 4, 16 or 64");
  require(link.pilot_spacing >= 1 && link.F >= link.pilot_spacing, "pilot spacing must fit the subcarrier count");
  require(link.n_pilot_symbols >= 0 && link.n_pilot_symbols <= 8, "at most 8 pilot symbols");
  const int T = link.T, F = link.F, L = link.n_taps;
  h->nb = link.mod_order == 4 ? 2 : link.mod_order == 16 ? 4 : 6;
  // pilots.cpp:13-31: "PILOT"-seeded Rng (splitmix64 -> mt19937_64), QPSK from two bits per pilot
  std::mt19937_64 rng(splitmix64(0x50494C4F54ull));
  h->pmask.assign(static_cast<size_t>(T) * F, 0);
  h->pvals.assign(static_cast<size_t>(T) * F * 2, 0.f);
  for (int k = 0; k < link.n_pilot_symbols; ++k) {
    const int t = link.pilot_symbols[k];
    require(t >= 0 && t < T, "pilot symbol index out of range");
    for (int f = 0; f < F; f += link.pilot_spacing) {
      const uint64_t b0 = rng() >> 63, b1 = rng() >> 63;
      const size_t i = static_cast<size_t>(t) * F + f;
      h->pmask[i] = 1;
      h->pvals[2 * i] = static_cast<float>((1.0 - 2.0 * static_cast<double>(b0)) / std::sqrt(2.0));
      h->pvals[2 * i + 1] = static_cast<float>((1.0 - 2.0 * static_cast<double>(b1)) / std::sqrt(2.0));
    }
  }
  // tap profile exactly as slots.tdl_response chooses it
  double spacing = link.tap_spacing_s;
  if (spacing <= 0) spacing = link.rms_delay_s > 0 ? link.rms_delay_s / 3.0 : 1.0 / (F * link.scs_hz);
  std::vector<double> p;
  if (link.rms_delay_s > 0) {
    p = tap_powers(link.rms_delay_s, spacing, L);
  } else {
    p.resize(static_cast<size_t>(L));
    double s = 0;
    for (int l = 0; l < L; ++l) s += (p[static_cast<size_t>(l)] = std::exp(-static_cast<double>(l)));
    for (double& v : p) v /= s;
  }
  h->gain.resize(static_cast<size_t>(L));
  h->tau.resize(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) {
    h->gain[static_cast<size_t>(l)] = static_cast<float>(std::sqrt(p[static_cast<size_t>(l)] / kSin));
    h->tau[static_cast<size_t>(l)] = l * spacing;
  }
}


void slot_noise_var(const cnrx_link& link, int64_t B, uint64_t seed, uint64_t slot0, float* out) {
  for (int64_t b = 0; b < B; ++b) {
    const uint64_t slot = slot0 + static_cast<uint64_t>(b);
    const U4 ws = philox(0u, P_SLOT, static_cast<uint32_t>(slot), static_cast<uint32_t>(slot >> 32),
                         static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    // same float arithmetic as re_kernel
    const float snr = static_cast<float>(link.snr_db_lo + (link.snr_db_hi - link.snr_db_lo) * static_cast<double>(unif(ws.x)));
    float v = std::pow(10.f, -snr / 10.f);
    if (link.has_interferer) {
      const float sir = static_cast<float>(link.sir_db_lo + (link.sir_db_hi - link.sir_db_lo) * static_cast<double>(unif(ws.z)));
      v += std::pow(10.f, -sir / 10.f);
    }
    out[b] = v;
  }
}

void slotgen_launch(const SlotGenArgs& a, float2* taps, float2* y, uint8_t* bits, float2* h, cudaStream_t s) {
  const int nch = a.has_interferer ? 2 : 1;
  const int64_t nt = a.B * nch * a.T * a.N * a.L;
  taps_kernel<<<static_cast<unsigned>(std::min<int64_t>((nt + 255) / 256, 148 * 16)), 256, 0, s>>>(a, taps);
  CNRX_CUDA(cudaGetLastError());
  const int64_t nre = a.B * a.T * a.F;
  re_kernel<<<static_cast<unsigned>(std::min<int64_t>((nre + 255) / 256, 148 * 32)), 256, 0, s>>>(a, taps, y, bits, h);
  CNRX_CUDA(cudaGetLastError());
}

void ber_launch(const float* llr, const uint8_t* bits, const uint8_t* data_mask, int64_t B, int64_t per_slot, int nb,
                unsigned long long* errors, cudaStream_t s) {
  CNRX_CUDA(cudaMemsetAsync(errors, 0, static_cast<size_t>(B) * sizeof(unsigned long long), s));
  const unsigned gx = static_cast<unsigned>(std::min<int64_t>((per_slot + 255) / 256, 64));
  ber_kernel<<<dim3(gx, static_cast<unsigned>(B)), 256, 0, s>>>(llr, bits, data_mask, per_slot, nb, errors);
  CNRX_CUDA(cudaGetLastError());
}

}  // namespace cnrx
