// conv_x3.cu — split-precision 3x3 / 1x1 "same" convolution on the sm_100a tensor cores: fp32-grade
// results (LLRs within 1e-4 relative of the reference's fp32 forward) at tensor-core rates.
//
// Replaces conetrx::conv2d (reference kernels.hpp:47-91) together with the nodes the plan compiler
// fuses into its epilogue — folded eval BN (norms.hpp:81-95 via network.hpp:458-459), ReLU
// (kernels.hpp:305), the residual add (network.hpp:463) and the next block's pre-activation
// (network.hpp:455-457) as a second output — for CNRX_BF16X3 / CNRX_FP16X3 plans (conv_x3.h).
//
// Every value v is carried as hi = round16(v), lo = round16(v - hi); weights likewise.  Per K-step
// of 16 channels the MMA warp issues two UMMAs (M = 128 plane rows, K = 16):
//     [D | E] += A_hi * [W_hi | W_lo]      (N = 2*Cout: the tap image stacks W_hi and W_lo rows)
//      D      += A_lo * W_hi               (N = Cout)
// and the epilogue adds D + E: the three products hi*Whi + lo*Whi + hi*Wlo, 3x the 16-bit plan's
// tensor work, with the fp32 plane's bytes.  SS UMMAs at N = Cout read more shared memory per cycle
// than the SM delivers (A 4 KB + B 2 KB per 32-cycle 128x64x16), so stacking the hi / lo weights along
// N (one A read for two products) cuts the operand traffic per K-step from 18 KB to 14 KB (64 ch).
// The plane layout makes every 3x3 tap a constant row shift (common.h), so a tile's whole K loop reads
// ONE TMA-loaded window of 128 + 2*halo rows of hi and lo.
//
// Warp roles (persistent, 1 CTA/SM):
//   warp 0     TMA producer: one hi+lo window per tile into a `stages`-deep ring
//   warp 1     TMEM allocator + single-thread MMA issuer (taps x K/16 x 2 UMMAs per tile)
//   warp 2     weight loader: every tap once (resident: 64-channel convs, 147 KB) or, when the split
//              weights exceed shared memory (96 channels: 331 KB), the taps of every tile through a
//              ring of `nslots` tap slots (plain bulk copies of the pre-swizzled tap images, L2-resident)
//   last 1-2   input ReLU of each window pair in place when the conv's input is relu(plane) (relu_in):
//              the producing conv then writes one plane instead of y and relu(y)
//   warps 3..  epilogue, 2 (3 for 96 channels) warps per TMEM lane quadrant, each owning a 32-channel
//              slice of its 32 rows: TMEM -> registers -> bias / residual (hi + lo) / ReLU -> hi, lo to
//              the output plane(s); accumulators double-buffered (tile j's epilogue overlaps tile j+1's MMAs)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "conv_x3.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kBoxRows = 32;
// epilogue warps per TMEM lane quadrant and channels per epilogue warp
__host__ __device__ constexpr int epi_per_quadrant(int cout) { return cout == 96 ? 3 : 2; }
// input-ReLU warps (96 channels: one, to stay within 128 registers at 16 warps)
__host__ __device__ constexpr int relu_warps(int cout) { return cout == 96 ? 1 : 2; }
// warps: producer, MMA, weight loader, 4 * EH epilogue, input ReLU
__host__ __device__ constexpr int threads_of(int cout) { return 32 * (3 + 4 * epi_per_quadrant(cout) + relu_warps(cout)); }
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
constexpr uint32_t kSmemLimit = 227u * 1024u;

__host__ __device__ constexpr int ch0_of(int cin) { return cin > 64 ? 64 : cin; }
__host__ __device__ constexpr int ch1_of(int cin) { return cin > 64 ? cin - 64 : 0; }
__host__ __device__ constexpr uint32_t swz_mode(int rb) {
  return rb == 128 ? kSwizzle128 : rb == 64 ? kSwizzle64 : rb == 32 ? kSwizzle32 : kSwizzleNone;
}
__host__ __device__ inline uint32_t swz_off(int rb, uint32_t r, uint32_t c) {
  if (rb == 128) return r * 128u + ((c ^ (r & 7u)) << 4);
  if (rb == 64) return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4);
  if (rb == 32) return r * 32u + ((c ^ ((r >> 2) & 1u)) << 4);
  return r * static_cast<uint32_t>(rb) + (c << 4);
}
__host__ __device__ constexpr uint32_t a1024(uint32_t x) { return (x + 1023u) & ~1023u; }
// one tap of the split weight image: per K-chunk [W_hi rows | W_lo rows], COUT x chunk 16-bit values each
__host__ __device__ constexpr uint32_t tap_bytes(int cin, int cout) {
  return 2u * static_cast<uint32_t>(cout) * static_cast<uint32_t>(cin) * 2u;
}
// UMMA issue order (A/B builds: -DCNRX_X3_ORDER=n): 0 interleaved per K-step into [D | E]; 1 (default) the lo
// product into its own accumulator F (Cout <= 64: [D | E | F]; 96 channels have no TMEM for it and use 0);
// 2 per tap all A_hi UMMAs, then all A_lo UMMAs; 3 the lo product accumulated into E.  Measured
// (profiles/r02_x3_order_ab.log, cfg2 64-ch convs): 1 is 3-4 % faster than 0; 2 and 3 equal 0 -- UMMAs of
// different N into the same accumulator columns do not overlap in the tensor pipe.
#ifndef CNRX_X3_ORDER
#define CNRX_X3_ORDER 1
#endif
__host__ __device__ constexpr int x3_order(int cout) { return CNRX_X3_ORDER == 1 && cout > 64 ? 0 : CNRX_X3_ORDER; }
// accumulator stage width: [D | E] (+ F) = 2 (3) * Cout columns; two stages
__host__ __device__ constexpr int acc_cols(int cout) { return (x3_order(cout) == 1 ? 3 : 2) * cout; }
__host__ __device__ constexpr uint32_t tmem_cols(int cout) {
  return 2 * acc_cols(cout) <= 128 ? 128 : 2 * acc_cols(cout) <= 256 ? 256 : 512;
}

struct Lay {
  uint32_t win_off, stage_bytes, sub[4], par_off, bar_off, total;
};
__host__ __device__ inline Lay x3_layout(int cin, int cout, int stages, int win_alloc, int nslots) {
  Lay s{};
  const uint32_t b0 = static_cast<uint32_t>(win_alloc * ch0_of(cin) * 2);
  const uint32_t b1 = static_cast<uint32_t>(win_alloc * ch1_of(cin) * 2);
  s.win_off = a1024(static_cast<uint32_t>(nslots) * tap_bytes(cin, cout));
  s.sub[0] = 0;                       // hi, channels [0, 64)
  s.sub[1] = a1024(b0);               // hi, channels [64, cin)
  s.sub[2] = a1024(s.sub[1] + b1);    // lo, channels [0, 64)
  s.sub[3] = a1024(s.sub[2] + b0);    // lo, channels [64, cin)
  s.stage_bytes = a1024(s.sub[3] + b1);
  uint32_t off = s.win_off + static_cast<uint32_t>(stages) * s.stage_bytes;
  s.par_off = off;  // bias, s2, t2 (fp32)
  off += (3u * static_cast<uint32_t>(cout) * 4u + 15u) & ~15u;
  s.bar_off = off;
  s.total = off + 256 + 1024;  // barriers (<= 31) + the TMEM slot, alignment slack of the dynamic base
  return s;
}

// In-place ReLU of n 16-byte chunk pairs of a split window (hi chunk i at hi + 16 i, its lo chunk at the
// same offset of the lo buffer: same row, same swizzle position).  relu(hi + lo) = (hi, lo) where hi > 0
// and (0, 0) elsewhere: hi = round16(v) has the sign of v, so a 16-bit lane compare on hi (signed integer
// compare of a sign-magnitude format: positive non-zero <=> > 0) masks both halves.  Batches of 8 chunk
// pairs per lane keep the loads in flight before the first store.
template <int RB>
__device__ __forceinline__ void relu_pairs(uint32_t hi, uint32_t lo, int n, int lane) {
  for (int c0 = 0; c0 < n; c0 += 32 * RB) {
    uint4 h[RB], l[RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < n) {
        h[u] = lds128(hi + static_cast<uint32_t>(c) * 16u);
        l[u] = lds128(lo + static_cast<uint32_t>(c) * 16u);
      }
    }
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < n) {
        uint32_t* hp = reinterpret_cast<uint32_t*>(&h[u]);
        uint32_t* lp = reinterpret_cast<uint32_t*>(&l[u]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t m = __vcmpgts2(hp[k], 0u);
          hp[k] &= m;
          lp[k] &= m;
        }
        sts128(hi + static_cast<uint32_t>(c) * 16u, h[u]);
        sts128(lo + static_cast<uint32_t>(c) * 16u, l[u]);
      }
    }
  }
}

// v -> (hi, lo) 16-bit pairs for two channels
template <bool H>
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  hi = pack2<H>(a, b);
  const float2 f = unpack2<H>(hi);
  lo = pack2<H>(a - f.x, b - f.y);
}

template <int CIN, int COUT, int KS, bool F16>
__global__ void __launch_bounds__(threads_of(COUT), 1) conv_x3_kernel(const __grid_constant__ X3Launch L) {
  constexpr int CH0 = ch0_of(CIN), CH1 = ch1_of(CIN);
  constexpr int RB0 = CH0 * 2, RB1 = CH1 * 2;
  constexpr uint32_t SW0 = swz_mode(RB0), SW1 = swz_mode(RB1);
  constexpr int TAPS = KS * KS;
  constexpr uint32_t TAPB = tap_bytes(CIN, COUT);
  constexpr uint32_t TMEM_COLS = tmem_cols(COUT);
  constexpr uint32_t IDESC1 = idesc_e16_f32<F16>(128, COUT);      // A_lo * W_hi
  constexpr uint32_t IDESC2 = idesc_e16_f32<F16>(128, 2 * COUT);  // A_hi * [W_hi | W_lo]
  constexpr int EH = epi_per_quadrant(COUT), NEPI = 4 * EH, ECH = COUT / EH;
  static_assert(ECH % 16 == 0, "epilogue warps own whole 16-column TMEM slices");

  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_align1024(smem_dyn);
  const int S = L.stages, NS = L.nslots;
  const bool resident = NS == TAPS;
  const Lay lay = x3_layout(CIN, COUT, S, L.win_alloc, NS);
  float* s_bias = reinterpret_cast<float*>(smem + lay.par_off);
  float* s_s2 = s_bias + COUT;
  float* s_t2 = s_s2 + COUT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* full = bars;          // [S] window landed
  uint64_t* empty = full + S;     // [S] window consumed by the MMAs
  uint64_t* wfull = empty + S;    // [NS] weight tap landed
  uint64_t* wempty = wfull + NS;  // [NS] weight tap consumed (streamed mode)
  uint64_t* tfull = wempty + NS;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;   // [2] accumulator drained
  uint64_t* ready = tempty + 2;   // [S] window ReLU'd in place (relu_in)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ready + S);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int G = L.ngroups;
  const int g = blockIdx.x % G;
  const int local = blockIdx.x / G;
  const int nct = (static_cast<int>(gridDim.x) - g + G - 1) / G;
  const X3Group& grp = L.g[g];
  const int64_t n_tiles = L.geo.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int k = 0; k < NS; ++k) {
      mbar_init(&wfull[k], 1);
      mbar_init(&wempty[k], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], NEPI);
    }
    for (int s = 0; s < S; ++s) mbar_init(&ready[s], relu_warps(COUT));
    fence_barrier_init();
  }
  if (warp >= 3) {
    for (int c = threadIdx.x - 96; c < COUT; c += 32 * NEPI) {
      s_bias[c] = grp.bias[c];
      s_s2[c] = grp.s2 ? grp.s2[c] : 1.f;
      s_t2[c] = grp.t2 ? grp.t2[c] : 0.f;
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_trigger();

  if (warp == 2) {
    // ------------------------------ weight loader (weights are plan constants: no PDL wait) -----------
    if (lane == 0) {
      if (resident) {
        for (int tap = 0; tap < TAPS; ++tap) {
          mbar_arrive_expect_tx(&wfull[tap], TAPB);
          bulk_load(smem + static_cast<uint32_t>(tap) * TAPB, grp.wimg + static_cast<size_t>(tap) * TAPB, TAPB,
                    &wfull[tap]);
        }
      } else {
        uint32_t wi = 0;
        for (int64_t tile = local; tile < n_tiles; tile += nct)
          for (int tap = 0; tap < TAPS; ++tap, ++wi) {
            const uint32_t slot = wi % static_cast<uint32_t>(NS);
            mbar_wait_backoff<64>(&wempty[slot], ((wi / static_cast<uint32_t>(NS)) & 1u) ^ 1u);
            mbar_arrive_expect_tx(&wfull[slot], TAPB);
            bulk_load(smem + slot * TAPB, grp.wimg + static_cast<size_t>(tap) * TAPB, TAPB, &wfull[slot]);
          }
      }
    }
  } else if (warp == 0) {
    // ------------------------------ window producer ------------------------------
    pdl_wait();
    if (lane == 0) {
      prefetch_tmap(&grp.map[0]);
      prefetch_tmap(&grp.map[2]);
      const int nboxes = (128 + 2 * grp.halo + kBoxRows - 1) / kBoxRows;
      const uint32_t stage_tx = static_cast<uint32_t>(nboxes * kBoxRows * CIN * 2 * 2);
      int j = 0;
      long long tr_prod = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
        const int s = j % S;
        const long long tw0 = L.trace ? clock64() : 0;
        mbar_wait_backoff<64>(&empty[s], (static_cast<uint32_t>(j / S) & 1u) ^ 1u);
        if (L.trace) tr_prod += clock64() - tw0;
        mbar_arrive_expect_tx(&full[s], stage_tx);
        uint8_t* win = smem + lay.win_off + s * lay.stage_bytes;
        const int32_t r0 = static_cast<int32_t>(tile * 128 - grp.halo);
        for (int bx = 0; bx < nboxes; ++bx) {
          const int32_t rr = r0 + bx * kBoxRows;
          tma_load_2d(win + lay.sub[0] + bx * kBoxRows * RB0, &grp.map[0], &full[s], 0, rr);
          tma_load_2d(win + lay.sub[2] + bx * kBoxRows * RB0, &grp.map[2], &full[s], 0, rr);
          if (CH1) {
            tma_load_2d(win + lay.sub[1] + bx * kBoxRows * RB1, &grp.map[1], &full[s], 0, rr);
            tma_load_2d(win + lay.sub[3] + bx * kBoxRows * RB1, &grp.map[3], &full[s], 0, rr);
          }
        }
      }
      if (L.trace) atomicAdd(&L.trace[kTraceProdWaitEmpty], static_cast<unsigned long long>(tr_prod));
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer --------------------------------
    // The whole warp runs the loop (waits, bookkeeping and descriptor bases stay warp-uniform) and one
    // elected lane issues each tap's UMMAs: issued from a lane-0-only branch every UMMA was wrapped in
    // an ELECT / BRA.U.ANY loop and the issue alone took ~6400 cycles per tile (trace), twice the
    // tensor time.  Descriptors: 32-bit low words advanced by one add per UMMA (sm100.cuh umma_ss_lohi).
    const uint32_t dh0 = sdesc_hi(8 * RB0, SW0), dh1 = sdesc_hi(8 * RB1, SW1);
    const uint32_t w_lo = sdesc_lo(smem_u32(smem));
    const int32_t T1 = L.geo.T1;
    int32_t trow[TAPS];  // window row of each tap's A operand
#pragma unroll
    for (int tap = 0; tap < TAPS; ++tap)
      trow[tap] = grp.halo + (tap / KS - KS / 2) + (tap % KS - KS / 2) * grp.dil * T1;
    if (resident)
      for (int tap = 0; tap < TAPS; ++tap) mbar_wait(&wfull[tap], 0);
    uint32_t wi = 0;
    int j = 0;
    long long tr_full = 0, tr_tmem = 0, tr_issue = 0;
    const long long t_start = clock64();
    const unsigned long long g_start = L.trace ? globaltimer_ns() : 0;
    for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
      const int s = j % S;
      const int a = j & 1;
      const long long tm0 = L.trace ? clock64() : 0;
      mbar_wait(L.relu_in ? &ready[s] : &full[s], static_cast<uint32_t>(j / S) & 1u);
      const long long tm1 = L.trace ? clock64() : 0;
      mbar_wait(&tempty[a], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
      const long long tm2 = L.trace ? clock64() : 0;
      if (L.trace) {
        tr_full += tm1 - tm0;
        tr_tmem += tm2 - tm1;
      }
      tc_fence_after();
      const uint32_t wlo = sdesc_lo(smem_u32(smem + lay.win_off + s * lay.stage_bytes));
      const uint32_t ah0 = wlo + (lay.sub[0] >> 4), al0 = wlo + (lay.sub[2] >> 4);
      const uint32_t ah1 = wlo + (lay.sub[1] >> 4), al1 = wlo + (lay.sub[3] >> 4);
      const uint32_t d_tmem = tbase + static_cast<uint32_t>(a * acc_cols(COUT));
      constexpr int ORD = x3_order(COUT);
      const uint32_t f_tmem = ORD == 1 ? d_tmem + 2 * COUT : ORD == 3 ? d_tmem + COUT : d_tmem;  // A_lo * W_hi
#pragma unroll
      for (int tap = 0; tap < TAPS; ++tap) {
        const uint32_t slot = resident ? static_cast<uint32_t>(tap) : wi % static_cast<uint32_t>(NS);
        if (!resident) {
          mbar_wait(&wfull[slot], (wi / static_cast<uint32_t>(NS)) & 1u);
          tc_fence_after();
        }
        if (elect_one()) {
          const uint32_t wb = w_lo + slot * (TAPB >> 4);
          const uint32_t r0 = static_cast<uint32_t>(trow[tap] * (RB0 >> 4));
          if (ORD == 2) {
#pragma unroll
            for (int kk = 0; kk < CH0 / 16; ++kk)
              umma_ss_lohi(d_tmem, ah0 + r0 + 2 * kk, dh0, wb + 2 * kk, dh0, IDESC2, (tap | kk) != 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < CH0 / 16; ++kk)
              umma_ss_lohi(d_tmem, al0 + r0 + 2 * kk, dh0, wb + 2 * kk, dh0, IDESC1, 1u);
          } else {
#pragma unroll
            for (int kk = 0; kk < CH0 / 16; ++kk) {
              umma_ss_lohi(d_tmem, ah0 + r0 + 2 * kk, dh0, wb + 2 * kk, dh0, IDESC2, (tap | kk) != 0 ? 1u : 0u);
              umma_ss_lohi(f_tmem, al0 + r0 + 2 * kk, dh0, wb + 2 * kk, dh0, IDESC1,
                           ORD == 1 && (tap | kk) == 0 ? 0u : 1u);
            }
          }
          if (CH1) {
            const uint32_t r1 = static_cast<uint32_t>(trow[tap] * (RB1 >> 4));
            const uint32_t w1 = wb + ((2 * COUT * RB0) >> 4);
#pragma unroll
            for (int kk = 0; kk < CH1 / 16; ++kk) {
              umma_ss_lohi(d_tmem, ah1 + r1 + 2 * kk, dh1, w1 + 2 * kk, dh1, IDESC2, 1u);
              umma_ss_lohi(f_tmem, al1 + r1 + 2 * kk, dh1, w1 + 2 * kk, dh1, IDESC1, 1u);
            }
          }
          if (!resident) umma_commit(&wempty[slot]);  // tap slot free once these MMAs have read it
        }
        __syncwarp();
        if (!resident) ++wi;
      }
      if (elect_one()) {
        umma_commit(&empty[s]);   // window stage free
        umma_commit(&tfull[a]);   // accumulator ready for the epilogue
      }
      __syncwarp();
      if (L.trace) tr_issue += clock64() - tm2;
    }
    if (L.trace && lane == 0) {
      atomicAdd(&L.trace[kTraceTotal], static_cast<unsigned long long>(clock64() - t_start));
      trace_cta_window(L.trace, g_start);
      atomicAdd(&L.trace[kTraceMmaWaitFull], static_cast<unsigned long long>(tr_full));
      atomicAdd(&L.trace[kTraceMmaWaitTmem], static_cast<unsigned long long>(tr_tmem));
      atomicAdd(&L.trace[kTraceMmaIssue], static_cast<unsigned long long>(tr_issue));
      atomicAdd(&L.trace[kTraceTiles], static_cast<unsigned long long>(j));
    }
  } else if (warp >= 3 + NEPI) {
    // ------------------------------ input ReLU (relu_in) ----------------------
    // The window is the tensor core's A operand (async proxy): ReLU it in place with generic 16-byte
    // shared accesses, then fence them to the async proxy before releasing the stage to the MMA warp.
    if (L.relu_in) {
      const int nrows = (128 + 2 * grp.halo + kBoxRows - 1) / kBoxRows * kBoxRows;
      constexpr int RW = relu_warps(COUT);
      const int rw = warp - 3 - NEPI;  // this warp's share: rows [rw * nrows / RW, (rw + 1) * nrows / RW)
      const int r0 = rw * nrows / RW, r1 = (rw + 1) * nrows / RW;
      int j = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
        const int s = j % S;
        mbar_wait(&full[s], static_cast<uint32_t>(j / S) & 1u);
        const uint32_t win = smem_u32(smem + lay.win_off + s * lay.stage_bytes);
        relu_pairs<COUT == 96 ? 4 : 8>(win + lay.sub[0] + r0 * RB0, win + lay.sub[2] + r0 * RB0, (r1 - r0) * (CH0 / 8), lane);
        if (CH1)
          relu_pairs<COUT == 96 ? 4 : 8>(win + lay.sub[1] + r0 * RB1, win + lay.sub[3] + r0 * RB1, (r1 - r0) * (CH1 / 8), lane);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ready[s]);
      }
    }
  } else {
    // ------------------------------ epilogue (warps 3..) ---------------------
    // EH warps per TMEM lane quadrant (warp % 4), each owning ECH of the Cout channels of its 32 rows:
    // one warp per quadrant left the epilogue latency-bound (a single dependent instruction stream per
    // SM sub-partition: ~5000 cycles per tile with the MMAs switched off)
    pdl_wait();
    named_bar_sync(1, 32 * NEPI);  // s_bias / s_s2 / s_t2 visible to all epilogue warps
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int cb = ((warp - 3) / 4) * ECH;  // first channel of this warp
    const int row = q * 32 + lane;
    const PlaneGeom geo = L.geo;
    int j = 0;
    long long tr_ew = 0, tr_ework = 0;
    for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
      const int a = j & 1;
      const long long te0 = L.trace ? clock64() : 0;
      const int64_t p = tile * 128 + row;
      const __nv_bfloat16* rrow = grp.res ? grp.res + p * (2 * COUT) : nullptr;
      __nv_bfloat16* orow = grp.out ? grp.out + p * (2 * COUT) : nullptr;
      __nv_bfloat16* orow2 = grp.out2 ? grp.out2 + p * (2 * COUT) : nullptr;
      // the residual slices are fetched before the accumulator wait: their latency hides behind the MMAs
      u32x8 rh[ECH / 16], rl[ECH / 16];
      if (rrow) {
#pragma unroll
        for (int i = 0; i < ECH / 16; ++i) {
          rh[i] = ldg256(rrow + cb + 16 * i);
          rl[i] = ldg256(rrow + COUT + cb + 16 * i);
        }
      }
      const bool valid = geo.valid(p);
      mbar_wait_backoff<128>(&tfull[a], static_cast<uint32_t>(j >> 1) & 1u);  // polls cost smem issue
      tc_fence_after();
      const long long te1 = L.trace ? clock64() : 0;
      if (L.trace) tr_ew += te1 - te0;
      const uint32_t taddr = tbase + static_cast<uint32_t>(a * acc_cols(COUT) + cb) + (static_cast<uint32_t>(q * 32) << 16);
      uint32_t r[ECH], e[ECH];
#pragma unroll
      for (int i = 0; i < ECH / 16; ++i) {
        tmem_ld16(taddr + 16 * i, *reinterpret_cast<uint32_t(*)[16]>(&r[16 * i]));         // D: hi*Whi (+ lo*Whi)
        tmem_ld16(taddr + COUT + 16 * i, *reinterpret_cast<uint32_t(*)[16]>(&e[16 * i]));  // E: hi*Wlo
      }
      if constexpr (x3_order(COUT) == 1) {  // F: lo*Whi, folded into E
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < ECH / 16; ++i) {
          uint32_t f[16];
          tmem_ld16(taddr + 2 * COUT + 16 * i, f);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k)
            e[16 * i + k] = __float_as_uint(__uint_as_float(e[16 * i + k]) + __uint_as_float(f[k]));
        }
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&tempty[a]);
      float* lrow = nullptr;  // LLR head (3x3 output conv): fp32 [B,T,F,nb] rows of valid positions
      if (grp.llr && valid) {
        int32_t bb, tt, ff;
        geo.coords(p, bb, tt, ff);
        lrow = grp.llr + ((static_cast<int64_t>(bb) * geo.T + tt) * geo.F + ff) * grp.nb;
      }
#pragma unroll
      for (int hp = 0; hp < ECH / 16; ++hp) {
        const int c0 = cb + hp * 16;
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          v[i] = (__uint_as_float(r[hp * 16 + i]) + __uint_as_float(e[hp * 16 + i])) + s_bias[c0 + i];
        if (grp.llr) {
          if (lrow) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (c0 + i < grp.nb) lrow[c0 + i] = v[i];
          }
          continue;
        }
        if (rrow) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 h = unpack2<F16>(rh[hp].v[i]), l = unpack2<F16>(rl[hp].v[i]);
            v[2 * i] += h.x + l.x;  // hi + lo is exact in fp32
            v[2 * i + 1] += h.y + l.y;
          }
        }
        if (grp.relu) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        if (!valid) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (orow) {
          u32x8 oh, ol;
#pragma unroll
          for (int i = 0; i < 8; ++i) split2<F16>(v[2 * i], v[2 * i + 1], oh.v[i], ol.v[i]);
          stg256(orow + c0, oh);
          stg256(orow + COUT + c0, ol);
        }
        if (orow2) {
          u32x8 oh, ol;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float x0 = fmaxf(v[2 * i] * s_s2[c0 + 2 * i] + s_t2[c0 + 2 * i], 0.f);
            const float x1 = fmaxf(v[2 * i + 1] * s_s2[c0 + 2 * i + 1] + s_t2[c0 + 2 * i + 1], 0.f);
            split2<F16>(valid ? x0 : 0.f, valid ? x1 : 0.f, oh.v[i], ol.v[i]);
          }
          stg256(orow2 + c0, oh);
          stg256(orow2 + COUT + c0, ol);
        }
      }
      if (L.trace) tr_ework += clock64() - te1;
    }
    if (L.trace && warp == 3 && lane == 0) {
      atomicAdd(&L.trace[kTraceEpiWaitFull], static_cast<unsigned long long>(tr_ew));
      atomicAdd(&L.trace[kTraceEpiWork], static_cast<unsigned long long>(tr_ework));
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, TMEM_COLS);
}

template <int CIN, int COUT, int KS, bool F16>
const char* launch_t(const X3Launch& L, int num_sms, cudaStream_t stream) {
  auto kern = conv_x3_kernel<CIN, COUT, KS, F16>;
  const Lay lay = x3_layout(CIN, COUT, L.stages, L.win_alloc, L.nslots);
  if (lay.total > kSmemLimit) throw Error(3, "conv_x3: working set exceeds shared memory");
  ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(lay.total));
  const int64_t work = static_cast<int64_t>(L.ngroups) * L.geo.n_tiles;
  int grid = static_cast<int>(work < num_sms ? work : num_sms);
  if (grid < L.ngroups) grid = L.ngroups;
  launch_pdl(kern, dim3(grid), dim3(threads_of(COUT)), lay.total, stream, L);
  static char name[96];
  snprintf(name, sizeof name, "conv_x3_kernel<%d,%d,%d,%s>", CIN, COUT, KS, F16 ? "f16x3" : "bf16x3");
  return name;
}

using LaunchFn = const char* (*)(const X3Launch&, int, cudaStream_t);

// the same layer shapes as the 16-bit plans' generic kernel (conv_tc.cu): every graph the bf16 plan lowers
// also lowers to the split plan
#define CNRX_X3_CASES(X)                                                                                     \
  X(16, 32, 1) X(16, 32, 3) X(32, 32, 1) X(32, 32, 3) X(16, 64, 1) X(32, 64, 1) X(64, 64, 1) X(64, 64, 3)   \
  X(16, 96, 1) X(32, 96, 1) X(64, 96, 1) X(96, 96, 1) X(96, 96, 3) X(32, 64, 3) X(64, 32, 3) X(32, 96, 3)     \
  X(16, 64, 3) X(16, 96, 3) X(96, 32, 3) X(64, 32, 1) X(128, 64, 1)

LaunchFn find_launch(int cin, int cout, int ks, bool h) {
#define X(a, b, c) \
  if (cin == a && cout == b && ks == c) return h ? &launch_t<a, b, c, true> : &launch_t<a, b, c, false>;
  CNRX_X3_CASES(X)
#undef X
  return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    CNRX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p) throw Error(4, "cuTensorMapEncodeTiled not available");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

bool conv_x3_supported(int cin, int cout, int ks) { return find_launch(cin, cout, ks, false) != nullptr; }

size_t conv_x3_wimg_bytes(int cin, int cout, int ks) { return static_cast<size_t>(ks) * ks * tap_bytes(cin, cout); }

size_t conv_x3_smem_bytes(int cin, int cout, int ks, int stages, int win_alloc, int nslots) {
  (void)ks;
  return x3_layout(cin, cout, stages, win_alloc, nslots).total;
}

bool conv_x3_config(int cin, int cout, int ks, int win_alloc, int* stages, int* nslots) {
  const int taps = ks * ks;
  // resident weights with a double-buffered window, else a weight-tap ring (deeper first)
  const int tries[][2] = {{taps, 3}, {taps, 2}, {4, 2}, {3, 2}, {2, 2}, {2, 1}};
  for (const auto& t : tries) {
    if (t[0] > taps) continue;
    if (x3_layout(cin, cout, t[1], win_alloc, t[0]).total <= kSmemLimit) {
      *nslots = t[0];
      *stages = t[1];
      return true;
    }
  }
  return false;
}

void conv_x3_pack_weights(const float* w, int ks, int cin_real, int cout_real, const float* scale, int cin, int cout,
                          bool fp16, uint8_t* img) {
  const int ch0 = ch0_of(cin);
  const int rb0 = ch0 * 2, rb1 = ch1_of(cin) * 2;
  std::memset(img, 0, conv_x3_wimg_bytes(cin, cout, ks));
  for (int tap = 0; tap < ks * ks; ++tap) {
    uint8_t* tb = img + static_cast<size_t>(tap) * tap_bytes(cin, cout);
    for (int co = 0; co < cout; ++co)
      for (int ci = 0; ci < cin; ++ci) {
        float v = 0.f;
        if (co < cout_real && ci < cin_real) {
          v = w[(static_cast<size_t>(tap) * cin_real + ci) * cout_real + co];  // [kh,kw,Cin,Cout], kernels.hpp:32
          if (scale) v *= scale[co];
        }
        const uint16_t hi = e16_from_float_host(v, fp16);
        const uint16_t lo = e16_from_float_host(v - e16_to_float_host(hi, fp16), fp16);
        // chunk c: 2*COUT rows, W_hi for output channel co in row co, W_lo in row COUT + co
        uint8_t* base = tb;
        int rb = rb0, k = ci;
        if (ci >= ch0) {
          base = tb + static_cast<size_t>(2 * cout) * rb0;
          rb = rb1;
          k = ci - ch0;
        }
        const uint32_t c16 = static_cast<uint32_t>(k / 8), e2 = static_cast<uint32_t>(k % 8) * 2;
        std::memcpy(base + swz_off(rb, static_cast<uint32_t>(co), c16) + e2, &hi, 2);
        std::memcpy(base + swz_off(rb, static_cast<uint32_t>(cout + co), c16) + e2, &lo, 2);
      }
  }
}

void conv_x3_make_maps(const void* plane, int64_t nalloc, int cin, CUtensorMap* maps) {
  const int chs[2] = {ch0_of(cin), ch1_of(cin)};
  for (int part = 0; part < 2; ++part)      // hi, lo
    for (int c = 0; c < 2; ++c) {           // K-chunk
      CUtensorMap* m = &maps[part * 2 + c];
      if (chs[c] == 0 || !plane) {
        std::memset(m, 0, sizeof(CUtensorMap));
        continue;
      }
      const int rb = chs[c] * 2;
      const CUtensorMapSwizzle sw = rb == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                    : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                    : rb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(chs[c]), static_cast<cuuint64_t>(nalloc)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * cin) * 2};
      cuuint32_t box[2] = {static_cast<cuuint32_t>(chs[c]), static_cast<cuuint32_t>(kBoxRows)};
      cuuint32_t es[2] = {1, 1};
      void* base = const_cast<uint8_t*>(static_cast<const uint8_t*>(plane)) + (part * cin + (c == 0 ? 0 : chs[0])) * 2;
      CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(4, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    }
}

const char* conv_x3_launch(int cin, int cout, int ks, const X3Launch& L, int num_sms, cudaStream_t stream) {
  LaunchFn fn = find_launch(cin, cout, ks, L.fp16 != 0);
  if (!fn) throw Error(3, "no split-precision conv instantiation for cin=" + std::to_string(cin) + " cout=" +
                              std::to_string(cout) + " k=" + std::to_string(ks));
  return fn(L, num_sms, stream);
}

}  // namespace cnrx
