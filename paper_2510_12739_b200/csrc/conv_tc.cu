// conv_tc.cu — 3x3 / 1x1 "same" convolution over bf16 activation planes as an implicit GEMM on the
// sm_100a tensor cores (tcgen05.mma kind::f16, fp32 accumulators in TMEM, operands staged by TMA).
//
// Replaces conetrx::conv2d (reference kernels.hpp:47-91) for the CoNet-Rx subnetworks together with
// the nodes the plan compiler fuses into its epilogue: the folded eval batch norm after the conv
// (norms.hpp:81-95 via network.hpp:458-459), ReLU (kernels.hpp:305), the residual add
// (network.hpp:463) and the pre-activation of the next block (ReLU, or BN+ReLU for RB blocks,
// network.hpp:455-457) as a second output.
//
// GEMM mapping: M = 128 consecutive plane rows (grid positions), N = Cout,
// K = Cin per tap.  Because the plane layout turns every 3x3 tap into a constant row shift, the
// whole K loop of one tile reads a single TMA-loaded window of 128 + 2*halo rows; tap t's A operand
// is that window addressed `halo + off_t` rows in (the UMMA descriptor swizzle is address-based —
// pinned by tools/probes/umma_probe.cu).  Weights (all taps) stay resident in shared memory for the
// CTA's lifetime.
//
// Warp roles (192 threads, persistent, 1 CTA/SM):
//   warp 0     TMA producer: weights once, then one window per tile into a `stages`-deep ring
//   warp 1     TMEM allocator + single-thread MMA issuer (9 taps x K/16 UMMAs per tile)
//   warps 2-5  epilogue: TMEM -> registers -> bias/residual/ReLU -> bf16 rows to the output plane(s);
//              TMEM accumulators are double-buffered so tile j's epilogue overlaps tile j+1's MMAs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "conv_tc.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kBoxRows = 32;  // TMA box height; a window is ceil(rows/32) boxes

__host__ __device__ constexpr int chunk0_ch(int cin) { return cin > 64 ? 64 : cin; }
__host__ __device__ constexpr int chunk1_ch(int cin) { return cin > 64 ? cin - 64 : 0; }
__host__ __device__ constexpr uint32_t swz_of_rowbytes(int rb) {
  return rb == 128 ? kSwizzle128 : rb == 64 ? kSwizzle64 : rb == 32 ? kSwizzle32 : kSwizzleNone;
}
__host__ __device__ constexpr int tmem_cols_for(int cout) {
  return 2 * cout <= 32 ? 32 : 2 * cout <= 64 ? 64 : 2 * cout <= 128 ? 128 : 2 * cout <= 256 ? 256 : 512;
}
// byte offset of 16-byte chunk `c` of row `r` in a K-major swizzled tile with `rb`-byte rows
__host__ __device__ inline uint32_t swz_offset(int rb, uint32_t r, uint32_t c) {
  if (rb == 128) return r * 128u + ((c ^ (r & 7u)) << 4);
  if (rb == 64) return r * 64u + ((c ^ ((r >> 1) & 3u)) << 4);
  if (rb == 32) return r * 32u + ((c ^ ((r >> 2) & 1u)) << 4);
  return r * static_cast<uint32_t>(rb) + (c << 4);
}

struct SmemLayout {
  uint32_t w_off, win_off, win_stage_bytes, win_chunk1_off;
  uint32_t res_off, stg_off, par_off, bar_off, total;
};
__host__ __device__ constexpr bool staged_epi(int cin, int cout) { return cin <= 64 && cout <= 64; }
// flags: bit 0 = some group has a residual, bit 1 = some group writes a second output
__host__ __device__ inline SmemLayout smem_layout(int cin, int cout, int ks, int stages, int win_alloc, int flags) {
  SmemLayout s{};
  const uint32_t wbytes = static_cast<uint32_t>(ks * ks * cout * cin * 2);
  s.w_off = 0;
  s.win_off = (wbytes + 1023u) & ~1023u;
  const uint32_t c0 = static_cast<uint32_t>(win_alloc * chunk0_ch(cin) * 2);
  const uint32_t c1 = static_cast<uint32_t>(win_alloc * chunk1_ch(cin) * 2);
  s.win_chunk1_off = (c0 + 1023u) & ~1023u;
  s.win_stage_bytes = (s.win_chunk1_off + c1 + 1023u) & ~1023u;
  uint32_t off = s.win_off + static_cast<uint32_t>(stages) * s.win_stage_bytes;
  if (staged_epi(cin, cout)) {
    s.res_off = off;                                   // 2 x [128 rows][cout] residual tiles
    if (flags & 1) off += 2u * 128u * static_cast<uint32_t>(cout) * 2u;
    s.stg_off = off;                                   // 4 warps x 2 outputs x [32 rows][cout]
    off += 4u * 2u * 32u * static_cast<uint32_t>(cout) * 2u;
  }
  s.par_off = off;                                     // bias, s2, t2 (fp32)
  off += (3u * static_cast<uint32_t>(cout) * 4u + 15u) & ~15u;
  s.bar_off = off;
  s.total = s.bar_off + 256 + 1024;  // barriers + alignment slack for the dynamic smem base
  return s;
}

// 1x1 convs with few input channels (the stem) are epilogue-latency bound: let three CTAs share an SM.
#ifndef CNRX_STEM_CTAS
#define CNRX_STEM_CTAS 4
#endif
template <int CIN, int COUT, int KS>
constexpr int min_ctas() { return KS == 1 && CIN <= 32 && COUT <= 64 ? CNRX_STEM_CTAS : 1; }

template <int CIN, int COUT, int KS, bool F16>
__global__ void __launch_bounds__(192, min_ctas<CIN, COUT, KS>()) conv_tc_kernel(const __grid_constant__ TcLaunch L) {
  constexpr int CH0 = chunk0_ch(CIN), CH1 = chunk1_ch(CIN);
  constexpr int RB0 = CH0 * 2, RB1 = CH1 * 2;
  constexpr uint32_t SW0 = swz_of_rowbytes(RB0), SW1 = swz_of_rowbytes(RB1);
  constexpr int TAPS = KS * KS;
  constexpr uint32_t WBYTES = TAPS * COUT * CIN * 2;
  constexpr uint32_t TMEM_COLS = tmem_cols_for(COUT);
  constexpr uint32_t IDESC = idesc_e16_f32<F16>(128, COUT);
  constexpr bool STAGED = staged_epi(CIN, COUT);
  constexpr int ORB = COUT * 2;  // output row bytes (staged path: one swizzle chunk)

  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_align1024(smem_dyn);
  const SmemLayout lay = smem_layout(CIN, COUT, KS, L.stages, L.win_alloc, L.flags);
  uint8_t* sW = smem + lay.w_off;
  float* s_bias = reinterpret_cast<float*>(smem + lay.par_off);
  float* s_s2 = s_bias + COUT;
  float* s_t2 = s_s2 + COUT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* w_full = bars;                  // [1]
  uint64_t* full = bars + 1;                // [stages]
  uint64_t* empty = full + L.stages;        // [stages]
  uint64_t* tfull = empty + L.stages;       // [2]
  uint64_t* tempty = tfull + 2;             // [2]
  uint64_t* rfull = tempty + 2;             // [2] residual tile landed
  uint64_t* rempty = rfull + 2;             // [2] residual tile consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int G = L.ngroups;
  const int g = blockIdx.x % G;
  const int local = blockIdx.x / G;
  const int nct = (static_cast<int>(gridDim.x) - g + G - 1) / G;
  const TcGroup& grp = L.g[g];
  const int64_t n_tiles = L.geo.n_tiles;
  const bool has_res = grp.res != nullptr;

  if (threadIdx.x == 0) {
    mbar_init(w_full, 1);
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
      mbar_init(&rfull[a], 1);
      mbar_init(&rempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp >= 2) {  // epilogue parameters to shared memory
    for (int c = threadIdx.x - 64; c < COUT; c += 128) {
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
  pdl_wait();  // PDL: the prologue above overlapped the previous kernel's tail

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      long long tr_prod = 0;
      prefetch_tmap(&grp.map[0]);
      if (CH1) prefetch_tmap(&grp.map[1]);
      mbar_arrive_expect_tx(w_full, WBYTES);
      bulk_load(sW, grp.wimg, WBYTES, w_full);
      const int nboxes = (128 + 2 * grp.halo + kBoxRows - 1) / kBoxRows;
      const uint32_t stage_tx = static_cast<uint32_t>(nboxes * kBoxRows * CIN * 2);
      int j = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
        const int s = j % L.stages;
        const uint32_t k = static_cast<uint32_t>(j / L.stages);
        const long long tw0 = L.trace ? clock64() : 0;
        mbar_wait(&empty[s], (k & 1u) ^ 1u);
        if (L.trace) tr_prod += clock64() - tw0;
        mbar_arrive_expect_tx(&full[s], stage_tx);
        uint8_t* win = smem + lay.win_off + s * lay.win_stage_bytes;
        const int32_t r0 = static_cast<int32_t>(tile * 128 - grp.halo);
        for (int bx = 0; bx < nboxes; ++bx) {
          tma_load_2d(win + bx * kBoxRows * RB0, &grp.map[0], &full[s], 0, r0 + bx * kBoxRows);
          if (CH1) tma_load_2d(win + lay.win_chunk1_off + bx * kBoxRows * RB1, &grp.map[1], &full[s], 0,
                               r0 + bx * kBoxRows);
        }
        if (STAGED && has_res) {
          const int a = j & 1;
          mbar_wait(&rempty[a], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&rfull[a], 128u * ORB);
          uint8_t* rb = smem + lay.res_off + a * 128 * ORB;
          for (int bx = 0; bx < 4; ++bx)
            tma_load_2d(rb + bx * 32 * ORB, &grp.res_map, &rfull[a], 0, static_cast<int32_t>(tile * 128 + bx * 32));
        }
      }
      if (L.trace) atomicAdd(&L.trace[kTraceProdWaitEmpty], static_cast<unsigned long long>(tr_prod));
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer --------------------------------
    if (lane == 0) {
      long long tr_full = 0, tr_tmem = 0, tr_issue = 0;
      const long long t_start = clock64();
    const unsigned long long g_start = globaltimer_ns();
      mbar_wait(w_full, 0);
      tc_fence_after();
      const uint32_t sW_addr = smem_u32(sW);
      const int32_t T1 = L.geo.T1;
      int j = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
        const int s = j % L.stages;
        const int a = j & 1;
        const long long tm0 = L.trace ? clock64() : 0;
        mbar_wait(&full[s], static_cast<uint32_t>(j / L.stages) & 1u);
        const long long tm1 = L.trace ? clock64() : 0;
        mbar_wait(&tempty[a], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
        const long long tm2 = L.trace ? clock64() : 0;
        if (L.trace) {
          tr_full += tm1 - tm0;
          tr_tmem += tm2 - tm1;
        }
        tc_fence_after();
        const uint32_t win_addr = smem_u32(smem + lay.win_off + s * lay.win_stage_bytes);
        const uint32_t d_tmem = tbase + static_cast<uint32_t>(a * COUT);
        uint32_t acc = 0;
#pragma unroll 1
        for (int tap = 0; tap < TAPS; ++tap) {
          const int dt = tap / KS - KS / 2, df = tap % KS - KS / 2;
          const int row = grp.halo + dt + df * grp.dil * T1;
          const uint32_t a0 = win_addr + static_cast<uint32_t>(row * RB0);
          const uint32_t b0 = sW_addr + static_cast<uint32_t>(tap * COUT * CIN * 2);
#pragma unroll
          for (int kk = 0; kk < CH0 / 16; ++kk) {
            const uint64_t ad = make_sdesc(a0 + kk * 32, 8 * RB0, SW0, 0);
            const uint64_t bd = make_sdesc(b0 + kk * 32, 8 * RB0, SW0, 0);
            umma_f16(d_tmem, ad, bd, IDESC, acc);
            acc = 1;
          }
          if (CH1) {
            const uint32_t a1 = win_addr + lay.win_chunk1_off + static_cast<uint32_t>(row * RB1);
            const uint32_t b1 = b0 + static_cast<uint32_t>(COUT * RB0);
#pragma unroll
            for (int kk = 0; kk < CH1 / 16; ++kk) {
              const uint64_t ad = make_sdesc(a1 + kk * 32, 8 * RB1, SW1, 0);
              const uint64_t bd = make_sdesc(b1 + kk * 32, 8 * RB1, SW1, 0);
              umma_f16(d_tmem, ad, bd, IDESC, 1);
            }
          }
        }
        umma_commit(&empty[s]);   // window stage free once these MMAs have read it
        umma_commit(&tfull[a]);   // accumulator ready for the epilogue
        if (L.trace) tr_issue += clock64() - tm2;
      }
      if (L.trace) {
        atomicAdd(&L.trace[kTraceTotal], static_cast<unsigned long long>(clock64() - t_start));
      trace_cta_window(L.trace, g_start);
        atomicAdd(&L.trace[kTraceMmaWaitFull], static_cast<unsigned long long>(tr_full));
        atomicAdd(&L.trace[kTraceMmaWaitTmem], static_cast<unsigned long long>(tr_tmem));
        atomicAdd(&L.trace[kTraceMmaIssue], static_cast<unsigned long long>(tr_issue));
        atomicAdd(&L.trace[kTraceTiles], static_cast<unsigned long long>(j));
      }
    }
  } else {
    // ------------------------------ epilogue (warps 2..5) ---------------------
    asm volatile("bar.sync 1, 128;" ::: "memory");  // s_bias / s_s2 / s_t2 visible to all epilogue warps
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = q * 32 + lane;
    const PlaneGeom geo = L.geo;
    uint8_t* stg = STAGED ? smem + lay.stg_off + q * 2 * 32 * ORB : nullptr;  // [out | out2] x [32][COUT]
    int j = 0;
    long long tr_ew = 0, tr_ework = 0;
    for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
      const int a = j & 1;
      // unstaged epilogue: this row's residual is fetched before waiting for the accumulator, so its
      // global-memory latency hides behind the tile's MMAs (one batch of COUT/8 16-byte loads)
      constexpr int NRES = STAGED ? 1 : COUT / 16;  // 32-byte (16-channel) pieces
      u32x8 rres[NRES];
      if constexpr (!STAGED) {
        if (grp.res) {
          const __nv_bfloat16* rrow = grp.res + (tile * 128 + q * 32 + lane) * COUT;
#pragma unroll
          for (int i = 0; i < NRES; ++i) rres[i] = ldg256(rrow + 16 * i);
        }
      }
      const long long te0 = L.trace ? clock64() : 0;
      mbar_wait(&tfull[a], static_cast<uint32_t>(j >> 1) & 1u);
      const long long te1 = L.trace ? clock64() : 0;
      if (L.trace) tr_ew += te1 - te0;
      tc_fence_after();
      const int64_t p = tile * 128 + row;
      const bool valid = geo.valid(p);
      const uint32_t taddr = tbase + static_cast<uint32_t>(a * COUT) + (static_cast<uint32_t>(q * 32) << 16);
      if (grp.llr) {
        // LLR head (a 3x3 output conv, NetSpec.kernel = 3): fp32 LLRs of valid rows in the reference layout
        // [B,T,F,nb], straight from the accumulator (no plane, no rounding)
        float* dst = nullptr;
        if (valid) {
          int32_t bb, tt, ff;
          geo.coords(p, bb, tt, ff);
          dst = grp.llr + ((static_cast<int64_t>(bb) * geo.T + tt) * geo.F + ff) * grp.nb;
        }
#pragma unroll 1
        for (int cc = 0; cc < COUT / 32; ++cc) {
          uint32_t r[32];
          tmem_ld32(taddr + cc * 32, r);
          tmem_ld_wait();
          if (cc == COUT / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tempty[a]);
          }
          if (dst) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (cc * 32 + i < grp.nb) dst[cc * 32 + i] = __uint_as_float(r[i]) + s_bias[cc * 32 + i];
          }
        }
      } else if constexpr (STAGED) {
        const uint8_t* rrow = nullptr;
        if (has_res) {
          mbar_wait(&rfull[a], static_cast<uint32_t>(j >> 1) & 1u);
          rrow = smem + lay.res_off + a * 128 * ORB;
        }
        // staging buffer free?  Launches without a second output use the out2 half as a second buffer
        // (alternate tiles), so the wait covers the store issued two tiles ago, not the one just issued
        const bool dbl = (L.flags & 2) == 0;
        uint8_t* sb = dbl && (j & 1) ? stg + 32 * ORB : stg;
        if (lane == 0) {
          if (dbl)
            bulk_wait_read1();
          else
            bulk_wait_read0();
        }
        __syncwarp();
#pragma unroll 1
        for (int cc = 0; cc < COUT / 32; ++cc) {
          uint32_t r[32];
          tmem_ld32(taddr + cc * 32, r);
          tmem_ld_wait();
          if (cc == COUT / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tempty[a]);
          }
#pragma unroll
          for (int v8 = 0; v8 < 4; ++v8) {
            const int c0 = cc * 32 + v8 * 8;
            const uint32_t chunk = static_cast<uint32_t>(c0 / 8);
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[v8 * 8 + i]) + s_bias[c0 + i];
            if (rrow) {
              const uint4 rv = *reinterpret_cast<const uint4*>(rrow + swz_offset(ORB, static_cast<uint32_t>(row), chunk));
              const uint32_t* rp = reinterpret_cast<const uint32_t*>(&rv);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f = unpack2<F16>(rp[i]);
                v[2 * i] += f.x;
                v[2 * i + 1] += f.y;
              }
            }
            if (grp.relu) {
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
            }
            if (!valid) {
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = 0.f;
            }
            const uint32_t so = swz_offset(ORB, static_cast<uint32_t>(lane), chunk);
            {
              uint4 o;
              uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
              for (int i = 0; i < 4; ++i) op[i] = pack2<F16>(v[2 * i], v[2 * i + 1]);
              *reinterpret_cast<uint4*>(sb + so) = o;
            }
            if (grp.out2) {
              uint4 o;
              uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float x0 = fmaxf(v[2 * i] * s_s2[c0 + 2 * i] + s_t2[c0 + 2 * i], 0.f);
                const float x1 = fmaxf(v[2 * i + 1] * s_s2[c0 + 2 * i + 1] + s_t2[c0 + 2 * i + 1], 0.f);
                op[i] = pack2<F16>(valid ? x0 : 0.f, valid ? x1 : 0.f);
              }
              *reinterpret_cast<uint4*>(stg + 32 * ORB + so) = o;
            }
          }
        }
        if (has_res) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[a]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int32_t r0 = static_cast<int32_t>(tile * 128 + q * 32);
          tma_store_2d(&grp.out_map, sb, 0, r0);
          if (grp.out2) tma_store_2d(&grp.out2_map, stg + 32 * ORB, 0, r0);
          bulk_commit();
        }
      } else {
        __nv_bfloat16* orow = grp.out ? grp.out + p * COUT : nullptr;
        __nv_bfloat16* orow2 = grp.out2 ? grp.out2 + p * COUT : nullptr;
        const bool has_r = grp.res != nullptr;
#pragma unroll
        for (int cc = 0; cc < COUT / 32; ++cc) {
          uint32_t r[32];
          tmem_ld32(taddr + cc * 32, r);
          tmem_ld_wait();
          if (cc == COUT / 32 - 1) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tempty[a]);
          }
          // two 16-channel pieces per 32-column chunk, each stored with one 256-bit access
#pragma unroll
          for (int hp = 0; hp < 2; ++hp) {
            const int c0 = cc * 32 + hp * 16;
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[hp * 16 + i]) + s_bias[c0 + i];
            if (has_r) {
              const u32x8& rv = rres[(c0 / 16) < NRES ? c0 / 16 : 0];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float2 f = unpack2<F16>(rv.v[i]);
                v[2 * i] += f.x;
                v[2 * i + 1] += f.y;
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
              u32x8 o;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                o.v[i] = pack2<F16>(v[2 * i], v[2 * i + 1]);
              }
              stg256(orow + c0, o);
            }
            if (orow2) {
              u32x8 o;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float x0 = fmaxf(v[2 * i] * s_s2[c0 + 2 * i] + s_t2[c0 + 2 * i], 0.f);
                const float x1 = fmaxf(v[2 * i + 1] * s_s2[c0 + 2 * i + 1] + s_t2[c0 + 2 * i + 1], 0.f);
                o.v[i] = pack2<F16>(valid ? x0 : 0.f, valid ? x1 : 0.f);
              }
              stg256(orow2 + c0, o);
            }
          }
        }
      }
      if (L.trace) tr_ework += clock64() - te1;
    }
    if (STAGED && lane == 0) bulk_wait0();  // all output stores complete before the CTA retires
    if (L.trace && q == 0 && lane == 0) {
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
const char* launch_t(const TcLaunch& L, int num_sms, cudaStream_t stream) {
  auto kern = conv_tc_kernel<CIN, COUT, KS, F16>;
  const SmemLayout lay = smem_layout(CIN, COUT, KS, L.stages, L.win_alloc, L.flags);
  ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(lay.total));
  // Several CTAs per SM when shared memory and TMEM allow (small-K convs, e.g. the 1x1 stem, are
  // bound by their epilogue; more resident epilogue warps hide its latency chains).
  // (the occupancy API under-reports here, so count registers / shared memory / TMEM directly)
  static thread_local int regs = -1;
  if (regs < 0) {
    cudaFuncAttributes fa{};
    CNRX_CUDA(cudaFuncGetAttributes(&fa, kern));
    regs = fa.numRegs;
  }
  const int by_regs = 65536 / (192 * ((regs + 7) / 8 * 8));
  const int by_smem = static_cast<int>((228u * 1024u) / (lay.total + 2048u));
  const int by_tmem = static_cast<int>(512 / tmem_cols_for(COUT));
  int per_sm = by_regs < by_smem ? by_regs : by_smem;
  if (per_sm > by_tmem) per_sm = by_tmem;
  if (per_sm > min_ctas<CIN, COUT, KS>()) per_sm = min_ctas<CIN, COUT, KS>();
  if (per_sm < 1) per_sm = 1;
  const int64_t work = static_cast<int64_t>(L.ngroups) * L.geo.n_tiles;
  const int64_t slots = static_cast<int64_t>(num_sms) * per_sm;
  int grid = static_cast<int>(work < slots ? work : slots);
  if (grid < L.ngroups) grid = L.ngroups;
  if (L.trace) fprintf(stderr, "[trace] conv_tc %d CTAs/SM (regs %d, smem %u B), grid %d\n", per_sm, regs, lay.total, grid);
  launch_pdl(kern, dim3(grid), dim3(192), lay.total, stream, L);
  static char name[96];
  snprintf(name, sizeof name, "conv_tc_kernel<%d,%d,%d%s>", CIN, COUT, KS, F16 ? ",f16" : "");
  return name;
}

using LaunchFn = const char* (*)(const TcLaunch&, int, cudaStream_t);

#define CNRX_TC_CASES(X)                                                                                     \
  X(16, 32, 1) X(16, 32, 3) X(32, 32, 1) X(32, 32, 3) X(16, 64, 1) X(32, 64, 1) X(64, 64, 1) X(64, 64, 3)   \
  X(16, 96, 1) X(32, 96, 1) X(64, 96, 1) X(96, 96, 1) X(96, 96, 3) X(32, 64, 3) X(64, 32, 3) X(32, 96, 3)     \
  X(16, 64, 3) X(16, 96, 3) X(96, 32, 3) X(64, 32, 1) X(128, 64, 1)

LaunchFn find_launch(int cin, int cout, int ks, bool h) {
#define X(a, b, c) \
  if (cin == a && cout == b && ks == c) return h ? &launch_t<a, b, c, true> : &launch_t<a, b, c, false>;
  CNRX_TC_CASES(X)
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

bool conv_tc_supported(int cin, int cout, int ks) { return find_launch(cin, cout, ks, false) != nullptr; }

bool conv_tc_staged(int cin, int cout) { return staged_epi(cin, cout); }

void conv_tc_make_row_map(const void* plane, int64_t nalloc, int c, CUtensorMap* map) {
  std::memset(map, 0, sizeof(CUtensorMap));
  if (!plane) return;
  if (c > 64) throw Error(3, "row map supports <= 64 channels");
  const int rb = c * 2;
  const CUtensorMapSwizzle sw = rb == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : rb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(nalloc)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(c) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(c), 32u};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(plane), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(4, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

size_t conv_tc_smem_bytes(int cin, int cout, int ks, int stages, int win_alloc, int flags) {
  return smem_layout(cin, cout, ks, stages, win_alloc, flags).total;
}

size_t conv_tc_wimg_bytes(int cin, int cout, int ks) { return static_cast<size_t>(ks) * ks * cout * cin * 2; }

const char* conv_tc_launch(int cin, int cout, int ks, const TcLaunch& L, int num_sms, cudaStream_t stream) {
  LaunchFn fn = find_launch(cin, cout, ks, L.fp16 != 0);
  if (!fn) throw Error(3, "no tcgen05 conv instantiation for cin=" + std::to_string(cin) + " cout=" +
                              std::to_string(cout) + " k=" + std::to_string(ks));
  return fn(L, num_sms, stream);
}

void conv_tc_pack_weights(const float* w, int ks, int cin_real, int cout_real, const float* scale, int cin,
                          int cout, bool fp16, uint8_t* img) {
  const int ch0 = chunk0_ch(cin), ch1 = chunk1_ch(cin);
  const int rb0 = ch0 * 2, rb1 = ch1 * 2;
  std::memset(img, 0, conv_tc_wimg_bytes(cin, cout, ks));
  for (int tap = 0; tap < ks * ks; ++tap) {
    uint8_t* tb = img + static_cast<size_t>(tap) * cout * cin * 2;
    for (int co = 0; co < cout; ++co)
      for (int ci = 0; ci < cin; ++ci) {
        float v = 0.f;
        if (co < cout_real && ci < cin_real) {
          // reference weight layout [kh,kw,Cin,Cout] (kernels.hpp:32), tap = dt*kw + df
          v = w[(static_cast<size_t>(tap) * cin_real + ci) * cout_real + co];
          if (scale) v *= scale[co];
        }
        const uint16_t b = e16_from_float_host(v, fp16);
        uint8_t* base;
        int rb, k;
        if (ci < ch0) {
          base = tb;
          rb = rb0;
          k = ci;
        } else {
          base = tb + static_cast<size_t>(cout) * rb0;
          rb = rb1;
          k = ci - ch0;
        }
        const uint32_t off = swz_offset(rb, static_cast<uint32_t>(co), static_cast<uint32_t>(k / 8)) + (k % 8) * 2;
        std::memcpy(base + off, &b, 2);
      }
  }
  (void)ch1;
}

void conv_tc_make_maps(const void* plane, int64_t nalloc, int cin, int box_rows, CUtensorMap* maps) {
  const int chs[2] = {chunk0_ch(cin), chunk1_ch(cin)};
  for (int c = 0; c < 2; ++c) {
    if (chs[c] == 0 || !plane) {
      std::memset(&maps[c], 0, sizeof(CUtensorMap));
      continue;
    }
    const int rb = chs[c] * 2;
    const CUtensorMapSwizzle sw = rb == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : rb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : rb == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                             : CU_TENSOR_MAP_SWIZZLE_NONE;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(chs[c]), static_cast<cuuint64_t>(nalloc)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cin) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(chs[c]), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    void* base = const_cast<uint8_t*>(static_cast<const uint8_t*>(plane)) + (c == 0 ? 0 : chs[0] * 2);
    CUresult r = encode_fn()(&maps[c], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(4, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  }
}

}  // namespace cnrx
