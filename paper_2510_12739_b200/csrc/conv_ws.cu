// conv_ws.cu — weights-stationary 3x3 conv (Cin = Cout = 64) on tcgen05 with A in TMEM.
//
// Same math as conv_tc.cu (replaces conetrx::conv2d, kernels.hpp:47-91, with the folded BN / ReLU /
// residual / next-block pre-activation epilogue), different GEMM orientation, chosen from measurement
// (tools/probes/umma_probe.cu, profiles/r01_umma_probe*.log):
//   * activations as the A operand with N = Cout = 64 make every UMMA read 6 KB of shared memory per
//     48 cycles = the SM's whole shared-memory bandwidth (LSU traffic is starved to ~8 B/clk), so the
//     tensor pipe idles and the epilogue cannot overlap;
//   * here the WEIGHTS are the A operand, resident in TMEM for the CTA's lifetime, and the activation
//     window is the B operand with N = 128 plane rows.  A-in-TMEM UMMAs run at the full 64 cycles for
//     128x128x16 and leave ~70 B/clk of shared memory for TMA and the epilogue.
// M = 128 lanes hold TWO 3x3 taps x 64 output channels, interleaved (lane 2c = tap A channel c, lane
// 2c+1 = tap B channel c) so the two partial sums of a channel sit in adjacent lanes of one warp.  The
// taps of a pair differ by one symbol (dt, dt+1) at the same frequency offset, i.e. by exactly one
// plane row, so tap B's partial sum for output row q is in accumulator column q+1: every output row
// q in [p0, p0+127) is A[q-p0] + B[q-p0+1].  Pairs: (dt=-1,0) for df in {-1,0,1} and (dt=+1, zero) for
// df in {-1,0,1} -> 6 UMMAs per 16-channel K step, 24 per tile, 75% of the issued MACs useful.
//
// Warp roles (576 threads, persistent, 1 CTA/SM, TMEM: 224 weight/identity columns + 2 x 128 accumulator):
//   warp 0     TMA producer: activation windows (4-stage ring) + residual tiles (2-deep ring)
//   warp 1     TMEM allocator + MMA issuer
//   warps 2-17 weights -> TMEM at start (2-5); epilogue in two groups of eight warps, one per
//              accumulator stage (alternate tiles): TMEM -> registers, lane-pair shuffle combine,
//              bias / ReLU / validity, bf16 pack, 8x8 lane-butterfly transpose so every lane writes
//              16-byte rows (8 channels of one plane row) to swizzled smem, TMA store of 127 rows.
// The residual add is done by the tensor core: an identity A block (TMEM columns 192..223) times
// the TMA-loaded residual tile accumulates R[p][c] into lane 2c, so the epilogue never reads it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "conv_tc.h"
#include "conv_ws.h"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kC = 64;            // channels in and out
constexpr int kRB = 128;          // bytes per plane row
constexpr int kTileRows = 127;    // output rows per tile
constexpr int kN = 128;           // UMMA N (plane rows per instruction)
constexpr int kPairs = 6;
constexpr int kKSteps = kC / 16;  // 4
constexpr int kWCols = kPairs * kKSteps * 8;  // 192 TMEM columns of weights
constexpr int kIdCol = kWCols;                // identity block for the residual: 4 K steps x 8 columns
constexpr int kAcc0 = 256;        // accumulator columns [256,384) and [384,512)
constexpr int kBox = 32;

struct WsLayout {
  uint32_t win_off, win_stage, res_off, stg_off, par_off, bar_off, total;
};
__host__ __device__ inline WsLayout ws_layout(int stages, int win_alloc) {
  WsLayout s{};
  s.win_off = 0;
  s.win_stage = static_cast<uint32_t>(win_alloc * kRB);  // multiple of 4 KB (32-row boxes)
  uint32_t off = s.win_stage * static_cast<uint32_t>(stages);
  s.res_off = off;                       // 2 x [128 rows][128 B]
  off += 2u * 128u * kRB;
  s.stg_off = off;                       // per epilogue group: [out | out2] x [128 rows][128 B]
  off += 2u * 2u * 128u * kRB;
  s.par_off = off;                       // bias, s2, t2
  off += 3u * kC * 4u;
  s.bar_off = off;
  s.total = off + 256 + 1024;
  return s;
}

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte_in_row) {
  return row * 128u + ((((byte_in_row >> 4) ^ (row & 7u)) << 4) | (byte_in_row & 15u));
}

// named barrier of one 256-thread epilogue group (constant ids: a register id makes ptxas reserve all 16)
__device__ __forceinline__ void epi_group_sync(int e) {
  if (e == 0) asm volatile("bar.sync 1, 256;" ::: "memory");
  else asm volatile("bar.sync 2, 256;" ::: "memory");
}

__global__ void __launch_bounds__(576, 1) conv_ws64_kernel(const __grid_constant__ WsLaunch L) {
  constexpr uint32_t IDESC = idesc_bf16_f32(128, kN);
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_dyn) + 1023) & ~uintptr_t(1023));
  const WsLayout lay = ws_layout(L.stages, L.win_alloc);
  float* s_bias = reinterpret_cast<float*>(smem + lay.par_off);
  float* s_s2 = s_bias + kC;
  float* s_t2 = s_s2 + kC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* full = bars;                  // [stages]
  uint64_t* empty = full + L.stages;      // [stages]
  uint64_t* tfull = empty + L.stages;     // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint64_t* rfull = tempty + 2;           // [2]
  uint64_t* rempty = rfull + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int G = L.ngroups;
  const int g = blockIdx.x % G;
  const int local = blockIdx.x / G;
  const int nct = (static_cast<int>(gridDim.x) - g + G - 1) / G;
  const WsGroup& grp = L.g[g];
  const int64_t n_tiles = L.n_tiles;
  const bool has_res = grp.res_map_valid != 0;
  const bool has_out2 = grp.out2_map_valid != 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
      mbar_init(&rfull[a], 1);
      mbar_init(&rempty[a], 1);
    }
    fence_barrier_init();
  }
  if (warp >= 2) {
    for (int c = threadIdx.x - 64; c < kC; c += 512) {
      s_bias[c] = grp.bias[c];
      s_s2[c] = grp.s2 ? grp.s2[c] : 1.f;
      s_t2[c] = grp.t2 ? grp.t2[c] : 0.f;
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp >= 2 && warp < 6) {
    // weights -> TMEM: block b = pair*4 + kstep occupies columns [8b, 8b+8); lane = packed row
    const int q = warp & 3;
    const uint32_t* src = grp.wimg + (static_cast<size_t>(q * 32 + lane) * 8);
#pragma unroll 1
    for (int b = 0; b < kPairs * kKSteps; ++b) {
      uint32_t r[8];
      const uint4* p4 = reinterpret_cast<const uint4*>(src + static_cast<size_t>(b) * 128 * 8);
      const uint4 v0 = p4[0], v1 = p4[1];
      r[0] = v0.x; r[1] = v0.y; r[2] = v0.z; r[3] = v0.w;
      r[4] = v1.x; r[5] = v1.y; r[6] = v1.z; r[7] = v1.w;
      tmem_st8(tbase + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(b * 8), r);
    }
    // identity (residual) block: lane 2c has a 1.0 at K index c
    const int Ln = q * 32 + lane;
#pragma unroll 1
    for (int kk = 0; kk < kKSteps; ++kk) {
      uint32_t r[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) r[e] = 0;
      if ((Ln & 1) == 0) {
        const int c = Ln >> 1;
        if (c / 16 == kk) {
          const int k = c % 16;
          r[k / 2] = 0x3F80u << ((k & 1) * 16);  // bf16 1.0
        }
      }
      tmem_st8(tbase + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(kIdCol + kk * 8), r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      prefetch_tmap(&grp.in_map);
      const int nboxes = (kN + 1 + 2 * grp.halo + kBox - 1) / kBox;
      const uint32_t stage_tx = static_cast<uint32_t>(nboxes * kBox * kRB);
      long long tr_prod = 0;
      int j = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
        const int s = j % L.stages;
        const uint32_t k = static_cast<uint32_t>(j / L.stages);
        const int64_t p0 = tile * kTileRows;
        const long long tp0 = L.trace ? clock64() : 0;
        mbar_wait(&empty[s], (k & 1u) ^ 1u);
        if (L.trace) tr_prod += clock64() - tp0;
        mbar_arrive_expect_tx(&full[s], stage_tx);
        uint8_t* win = smem + lay.win_off + s * lay.win_stage;
        const int32_t r0 = static_cast<int32_t>(p0 - grp.halo);
        for (int bx = 0; bx < nboxes; ++bx)
          tma_load_2d(win + bx * kBox * kRB, &grp.in_map, &full[s], 0, r0 + bx * kBox);
        if (has_res) {
          const int a = j & 1;
          const long long tp1 = L.trace ? clock64() : 0;
          mbar_wait(&rempty[a], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
          if (L.trace) tr_prod += clock64() - tp1;
          mbar_arrive_expect_tx(&rfull[a], 128u * kRB);
          uint8_t* rb = smem + lay.res_off + a * 128 * kRB;
          for (int bx = 0; bx < 4; ++bx)
            tma_load_2d(rb + bx * kBox * kRB, &grp.res_map, &rfull[a], 0, static_cast<int32_t>(p0 + bx * kBox));
        }
      }
      if (L.trace) atomicAdd(&L.trace[kTraceProdWaitEmpty], static_cast<unsigned long long>(tr_prod));
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer --------------------------------
    // pair p: A-half tap (dt = -1 or +1, df), B-half tap dt + 1 (real for the first three pairs)
    int32_t shift[kPairs];
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
      const int df = p % 3 - 1;
      const int dt = p < 3 ? -1 : 1;
      shift[p] = grp.halo + dt + df * grp.dil * L.geo.T1;
    }
    long long tr_full = 0, tr_tmem = 0, tr_issue = 0;
    const long long t_start = clock64();
    int j = 0;
    for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
      const int s = j % L.stages;
      const int a = j & 1;
      const long long tm0 = clock64();
      mbar_wait(&full[s], static_cast<uint32_t>(j / L.stages) & 1u);
      const long long tm1 = clock64();
      mbar_wait(&tempty[a], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
      const long long tm2 = clock64();
      tr_full += tm1 - tm0;
      tr_tmem += tm2 - tm1;
      tc_fence_after();
      if (elect_one()) {
        const uint32_t win_addr = smem_u32(smem + lay.win_off + s * lay.win_stage);
        const uint32_t d_tmem = tbase + kAcc0 + static_cast<uint32_t>(a * kN);
        const uint64_t bdesc0 = make_sdesc(win_addr, 8 * kRB, kSwizzle128, 0);
#pragma unroll
        for (int p = 0; p < kPairs; ++p) {
#pragma unroll
          for (int kk = 0; kk < kKSteps; ++kk) {
            const uint64_t bd = bdesc0 + static_cast<uint64_t>((shift[p] * kRB + kk * 32) >> 4);
            umma_bf16_ts(d_tmem, tbase + static_cast<uint32_t>((p * kKSteps + kk) * 8), bd, IDESC,
                         (p | kk) != 0 ? 1u : 0u);
          }
        }
        if (has_res) {
          mbar_wait(&rfull[a], static_cast<uint32_t>(j >> 1) & 1u);
          tc_fence_after();
          const uint64_t rdesc0 = make_sdesc(smem_u32(smem + lay.res_off + a * 128 * kRB), 8 * kRB, kSwizzle128, 0);
#pragma unroll
          for (int kk = 0; kk < kKSteps; ++kk)
            umma_bf16_ts(d_tmem, tbase + static_cast<uint32_t>(kIdCol + kk * 8),
                         rdesc0 + static_cast<uint64_t>((kk * 32) >> 4), IDESC, 1u);
          umma_commit(&rempty[a]);
        }
        umma_commit(&empty[s]);
        umma_commit(&tfull[a]);
      }
      __syncwarp();
      tr_issue += clock64() - tm2;
    }
    if (L.trace && lane == 0) {
      atomicAdd(&L.trace[kTraceTotal], static_cast<unsigned long long>(clock64() - t_start));
      atomicAdd(&L.trace[kTraceMmaWaitFull], static_cast<unsigned long long>(tr_full));
      atomicAdd(&L.trace[kTraceMmaWaitTmem], static_cast<unsigned long long>(tr_tmem));
      atomicAdd(&L.trace[kTraceMmaIssue], static_cast<unsigned long long>(tr_issue));
      atomicAdd(&L.trace[kTraceTiles], static_cast<unsigned long long>(j));
    }
  } else {
    // ------------------------------ epilogue (warps 2..17) --------------------
    // Two groups of eight warps, group e owning accumulator stage e (tiles j with j % 2 == e), so one
    // group's TMEM reads overlap the other group's shared-memory writes and TMA stores.  In a group,
    // warp (q, H) covers TMEM lane quadrant q and accumulator columns [64H, 64H + 64) as two 32-column
    // chunks.
    const int e = (warp - 2) >> 3;     // epilogue group == accumulator stage
    const int q = warp & 3;            // TMEM lane quadrant
    const int H = ((warp - 2) >> 2) & 1;
    const int Ln = q * 32 + lane;      // accumulator lane
    const int co = Ln >> 1;            // output channel of this lane
    const bool odd = (lane & 1) != 0;  // B-half lane
    const int idx = (lane >> 1) & 7;   // position in the 8-lane transpose group (same parity, same half-warp)
    const int c0 = q * 16 + (lane >> 4) * 8;  // first of the 8 channels this lane writes after the transpose
    const PlaneGeom geo = L.geo;
    uint8_t* stg = smem + lay.stg_off + e * 2 * 128 * kRB;
    const float bias = s_bias[co];
    const bool relu2_only = grp.s2 == nullptr;
    const bool lead = ((warp - 2) & 7) == 0 && lane == 0;
    long long tr_ew = 0, tr_comb = 0, tr_sw = 0, tr_wr = 0;
    int j = e;
    for (int64_t tile = local + static_cast<int64_t>(e) * nct; tile < n_tiles; tile += 2 * static_cast<int64_t>(nct), j += 2) {
      const int64_t p0 = tile * kTileRows;
      const long long te0 = clock64();
      mbar_wait(&tfull[e], static_cast<uint32_t>(j >> 1) & 1u);
      const long long te1 = clock64();
      tr_ew += te1 - te0;
      tc_fence_after();
      // chunk h (accumulator columns 64H + 32h .. +31, plus the next column): row 64H + 32h + k is
      // A[k] + B[k+1]; even lanes finalise k in [0,16), odd lanes k in [16,32).  pk[h][i] packs rows
      // (2i, 2i+1) of this lane's 16 rows, channel co.  The stage is released after the second load.
      const uint32_t taddr = tbase + kAcc0 + static_cast<uint32_t>(e * kN + 64 * H) + (static_cast<uint32_t>(q * 32) << 16);
      uint32_t pk[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t ra[32], rx[1];
        tmem_ld32(taddr + 32 * h, ra);
        if (H == 0 || h == 0) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(rx[0]) : "r"(taddr + 32 * h + 32) : "memory");
        } else {
          rx[0] = 0;
        }
        tmem_ld_wait();
        if (h == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[e]);
        }
#define CNRX_R(i) ((i) < 32 ? ra[(i) & 31] : rx[0])
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          const uint32_t send = odd ? CNRX_R(m + 1) : CNRX_R(16 + m);
          const float recv = __uint_as_float(__shfl_xor_sync(0xffffffffu, send, 1));
          const float mine = __uint_as_float(odd ? CNRX_R(17 + m) : CNRX_R(m));
          float v = mine + recv + bias;
          if (grp.relu) v = fmaxf(v, 0.f);
          const uint32_t hv = static_cast<uint32_t>(__bfloat16_as_ushort(__float2bfloat16_rn(v)));
          if ((m & 1) == 0) pk[h][m >> 1] = hv;
          else pk[h][m >> 1] |= hv << 16;
        }
#undef CNRX_R
      }
      // 8x8 transpose (16-bit elements) inside each group of 8 lanes (lane bits 1..3), per block of 8 rows:
      // afterwards pk[h][4b .. 4b+3] of lane idx = channels c0..c0+7 of row 64H + 32h + (odd ? 16 : 0) + 8b + idx.
#pragma unroll
      for (int hb = 0; hb < 4; ++hb) {
        uint32_t& r0 = pk[hb >> 1][4 * (hb & 1) + 0];
        uint32_t& r1 = pk[hb >> 1][4 * (hb & 1) + 1];
        uint32_t& r2 = pk[hb >> 1][4 * (hb & 1) + 2];
        uint32_t& r3 = pk[hb >> 1][4 * (hb & 1) + 3];
        {  // level 1: swap off-diagonal 4x4 blocks between idx and idx^4
          const bool lo = (idx & 4) == 0;
          const uint32_t s0 = lo ? r2 : r0, s1 = lo ? r3 : r1;
          const uint32_t g0 = __shfl_xor_sync(0xffffffffu, s0, 8), g1 = __shfl_xor_sync(0xffffffffu, s1, 8);
          if (lo) { r2 = g0; r3 = g1; } else { r0 = g0; r1 = g1; }
        }
        {  // level 2: swap off-diagonal 2x2 blocks between idx and idx^2
          const bool lo = (idx & 2) == 0;
          const uint32_t s0 = lo ? r1 : r0, s1 = lo ? r3 : r2;
          const uint32_t g0 = __shfl_xor_sync(0xffffffffu, s0, 4), g1 = __shfl_xor_sync(0xffffffffu, s1, 4);
          if (lo) { r1 = g0; r3 = g1; } else { r0 = g0; r2 = g1; }
        }
        {  // level 3: swap off-diagonal elements between idx and idx^1
          const bool lo = (idx & 1) == 0;
          const uint32_t g0 = __shfl_xor_sync(0xffffffffu, r0, 2), g1 = __shfl_xor_sync(0xffffffffu, r1, 2);
          const uint32_t g2 = __shfl_xor_sync(0xffffffffu, r2, 2), g3 = __shfl_xor_sync(0xffffffffu, r3, 2);
          r0 = lo ? __byte_perm(r0, g0, 0x5410) : __byte_perm(g0, r0, 0x7632);
          r1 = lo ? __byte_perm(r1, g1, 0x5410) : __byte_perm(g1, r1, 0x7632);
          r2 = lo ? __byte_perm(r2, g2, 0x5410) : __byte_perm(g2, r2, 0x7632);
          r3 = lo ? __byte_perm(r3, g3, 0x5410) : __byte_perm(g3, r3, 0x7632);
        }
      }
      const long long te2 = clock64();
      tr_comb += te2 - te1;
      // staging buffer free? (this group's previous TMA store has read it)
      if (lead) bulk_wait_read0();
      epi_group_sync(e);
      const long long te3 = clock64();
      tr_sw += te3 - te2;
#pragma unroll
      for (int hb = 0; hb < 4; ++hb) {
        const uint32_t row = static_cast<uint32_t>(64 * H + 32 * (hb >> 1) + (odd ? 16 : 0) + 8 * (hb & 1) + idx);
        const bool valid = geo.valid(p0 + row);  // row 127 is never stored
        const uint32_t* pr = &pk[hb >> 1][4 * (hb & 1)];
        uint4 o = make_uint4(pr[0], pr[1], pr[2], pr[3]);
        if (!valid) o = make_uint4(0, 0, 0, 0);
        const uint32_t off = row * 128u + (((static_cast<uint32_t>(c0 >> 3)) ^ (row & 7u)) << 4);
        *reinterpret_cast<uint4*>(stg + off) = o;
        if (has_out2) {
          uint4 u;
          if (relu2_only) {
            const __nv_bfloat162 z = __float2bfloat162_rn(0.f);
            __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&o);
            __nv_bfloat162* up = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) up[i] = __hmax2(op[i], z);
          } else {
            const __nv_bfloat162* op = reinterpret_cast<const __nv_bfloat162*>(&o);
            __nv_bfloat162* up = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __bfloat1622float2(op[i]);
              const float x0 = fmaxf(f.x * s_s2[c0 + 2 * i] + s_t2[c0 + 2 * i], 0.f);
              const float x1 = fmaxf(f.y * s_s2[c0 + 2 * i + 1] + s_t2[c0 + 2 * i + 1], 0.f);
              up[i] = __floats2bfloat162_rn(valid ? x0 : 0.f, valid ? x1 : 0.f);
            }
          }
          *reinterpret_cast<uint4*>(stg + 128 * kRB + off) = u;
        }
      }
      tr_wr += clock64() - te3;
      fence_proxy_async_smem();
      epi_group_sync(e);
      if (lead) {
        tma_store_2d(&grp.out_map, stg, 0, static_cast<int32_t>(p0));
        if (has_out2) tma_store_2d(&grp.out2_map, stg + 128 * kRB, 0, static_cast<int32_t>(p0));
        bulk_commit();
      }
    }
    if (lead) bulk_wait0();
    if (L.trace && lead && e == 0) {
      atomicAdd(&L.trace[kTraceEpiWaitFull], static_cast<unsigned long long>(tr_ew));
      atomicAdd(&L.trace[kWsTraceCombine], static_cast<unsigned long long>(tr_comb));
      atomicAdd(&L.trace[kWsTraceStageWait], static_cast<unsigned long long>(tr_sw));
      atomicAdd(&L.trace[kWsTraceWrite], static_cast<unsigned long long>(tr_wr));
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_ws() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    CNRX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr));
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void make_map(const void* plane, int64_t nalloc, uint32_t box_rows, CUtensorMap* m) {
  std::memset(m, 0, sizeof(CUtensorMap));
  if (!plane) return;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(kC), static_cast<cuuint64_t>(nalloc)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(kRB)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kC), box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn_ws()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(plane), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(4, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

}  // namespace

size_t conv_ws64_wimg_bytes() { return static_cast<size_t>(kPairs) * kKSteps * 128 * 8 * 4; }

void conv_ws64_pack_weights(const float* w, const float* scale, uint32_t* img) {
  // w: reference layout [3][3][64][64] = [dt+1][df+1][ci][co]; img: [block = pair*4 + kstep][lane][8 u32]
  std::memset(img, 0, conv_ws64_wimg_bytes());
  for (int p = 0; p < kPairs; ++p) {
    const int df = p % 3 - 1;
    const int dtA = p < 3 ? -1 : 1;
    for (int half = 0; half < 2; ++half) {
      const int dt = dtA + half;
      const bool real = half == 0 || p < 3;
      for (int co = 0; co < kC; ++co) {
        const int lane = 2 * co + half;
        for (int ci = 0; ci < kC; ++ci) {
          float v = 0.f;
          if (real) {
            v = w[((static_cast<size_t>(dt + 1) * 3 + (df + 1)) * kC + ci) * kC + co];
            if (scale) v *= scale[co];
          }
          const __nv_bfloat16 b = __float2bfloat16(v);
          uint16_t bits;
          std::memcpy(&bits, &b, 2);
          const int kk = ci / 16, e = ci % 16;
          uint32_t& word = img[((static_cast<size_t>(p) * kKSteps + kk) * 128 + lane) * 8 + e / 2];
          word |= static_cast<uint32_t>(bits) << ((e & 1) * 16);
        }
      }
    }
  }
}

void conv_ws64_make_maps(const void* in, const void* res, const void* out, const void* out2, int64_t nalloc,
                         WsGroup* g) {
  make_map(in, nalloc, kBox, &g->in_map);
  make_map(res, nalloc, kBox, &g->res_map);
  make_map(out, nalloc, kTileRows, &g->out_map);
  make_map(out2, nalloc, kTileRows, &g->out2_map);
  g->res_map_valid = res != nullptr;
  g->out2_map_valid = out2 != nullptr;
}

size_t conv_ws64_smem_bytes(int stages, int win_alloc) { return ws_layout(stages, win_alloc).total; }

int conv_ws64_win_alloc(int halo) { return (kN + 1 + 2 * halo + kBox - 1) / kBox * kBox; }

int64_t conv_ws64_tiles(int64_t nalloc) { return (nalloc + kTileRows - 1) / kTileRows; }

const char* conv_ws64_launch(const WsLaunch& L, int num_sms, cudaStream_t stream) {
  const WsLayout lay = ws_layout(L.stages, L.win_alloc);
  static thread_local int configured = -1;
  if (configured < static_cast<int>(lay.total)) {
    CNRX_CUDA(cudaFuncSetAttribute(conv_ws64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(lay.total)));
    configured = static_cast<int>(lay.total);
  }
  const int64_t work = static_cast<int64_t>(L.ngroups) * L.n_tiles;
  int grid = static_cast<int>(work < num_sms ? work : num_sms);
  if (grid < L.ngroups) grid = L.ngroups;
  conv_ws64_kernel<<<grid, 576, lay.total, stream>>>(L);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, conv_ws64_kernel);
    throw Error(4, std::string("conv_ws64 launch failed: ") + cudaGetErrorString(err) + " (regs " +
                       std::to_string(fa.numRegs) + ", max threads " + std::to_string(fa.maxThreadsPerBlock) +
                       ", static smem " + std::to_string(fa.sharedSizeBytes) + ", dynamic " +
                       std::to_string(lay.total) + ")");
  }
  return "conv_ws64_kernel";
}

}  // namespace cnrx
