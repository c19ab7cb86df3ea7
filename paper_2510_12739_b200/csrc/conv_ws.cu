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
// Warp roles (576 threads, persistent, 1 CTA/SM, TMEM: 192 weight columns + 2 x 128 accumulator):
//   warp 0     TMA producer: activation windows (4-stage ring); residual tiles are streamed by the
//              epilogue group that consumes them
//   warp 1     TMEM allocator + MMA issuer
//   warp 18    input ReLU of the window in shared memory when the plan asks for it (relu_in)
//   warps 2-17 weights -> TMEM at start (2-5); epilogue in two groups of eight warps, one per
//              accumulator stage (alternate tiles): TMEM -> registers, lane-pair shuffle combine,
//              bias / ReLU / validity, bf16 pack, 8x8 lane-butterfly transpose so every lane writes
//              16-byte rows (8 channels of one plane row) to swizzled smem, TMA store of 127 rows.
// With a residual the epilogue transposes the combined fp32 values (8x8 lane butterflies) so each
// lane holds 8 channels of one row, adds the TMA-staged residual row chunk with one 16-byte shared
// load, then rounds to bf16 (fp32 conv + bias + residual, a single rounding as the reference).
//
// Fused interaction + LLR head (kWsHead, opt-in CNRX_HEADFUSE=1): the subnetworks' last convs run as
// clusters of kNS CTAs (rank r = fold operand r) over the same tiles.  Each rank stages its bf16 output
// tile, copies the rows that rank d folds into d's receive slots (cp.async.bulk shared::cta ->
// shared::cluster), then folds its own third of the rows over all kNS tiles (head.cu's fp32 fold ->
// bf16 z), warp 18 runs the head as four UMMAs over the z rows (sm100.cuh head_tc_umma, the same
// instructions as head.cu, so the LLRs are bit-identical), and the LLRs are read from TMEM at the
// group's next tile.  The subnetworks' last activations never reach HBM.  Measured slower than conv +
// head kernel (cfg2: 1.02 ms vs 0.84 ms): the c2 epilogue has ~25 % slack per tile, and the exchange
// plus the fold pass and the LLR drain exceed it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "conv_tc.h"
#include "conv_ws.h"
#include "kernels.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kC = 64;            // channels in and out
constexpr int kRB = 128;          // bytes per plane row
constexpr int kTileRows = 127;    // output rows per tile
constexpr int kN = 128;           // UMMA N (plane rows per instruction)
constexpr int kPairs = 6;
constexpr int kKSteps = kC / 16;  // 4
constexpr int kAcc0 = 256;        // accumulator columns [256,384) and [384,512)
constexpr int kBox = 32;

struct WsLayout {
  uint32_t win_off, win_stage, res_off, stg_off, par_off, hw_off, fold_off, bar_off, total;
};
__host__ __device__ inline WsLayout ws_layout(int stages, int win_alloc, bool head = false) {
  WsLayout s{};
  s.win_off = 0;
  s.win_stage = static_cast<uint32_t>(win_alloc * kRB);  // multiple of 4 KB (32-row boxes)
  uint32_t off = s.win_stage * static_cast<uint32_t>(stages);
  s.res_off = off;                       // 2 groups x 2 buffers x [128 rows][128 B]
  off += 4u * 128u * kRB;
  s.stg_off = off;                       // per epilogue group: [out | out2] x [128 rows][128 B]
  off += 2u * 2u * 128u * kRB;
  s.par_off = off;                       // bias, s2, t2
  off += 3u * kC * 4u;
  s.hw_off = off;                        // fused head: bf16 head weight image (1024-aligned)
  s.fold_off = off;                      // fused head: fold scale / shift [3 steps][2][64] fp32
  if (head) {
    s.hw_off = (off + 1023u) & ~1023u;
    s.fold_off = s.hw_off + kHeadTcWBytes;
    off = s.fold_off + 3u * 2u * kC * 4u;
  }
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

// Epilogue variant flags (compile-time so the unrolled epilogue carries no per-element branches);
// kWsDynamic reads them from the launch instead.
enum : int { kWsRes = 1, kWsOut2 = 2, kWsOut2Bn = 4, kWsRelu = 8, kWsReluIn = 16, kWsHead = 32, kWsDynamic = -1 };
constexpr uint32_t kHeadCol = 192;  // fused head: TMEM columns [192, 256) = [2 groups][2 tiles][16] (free between weights and accumulators)
constexpr int kWsThreads = 640;  // 20 warps: producer, MMA (stage 0), 16 epilogue, input-ReLU, MMA (stage 1)

// Poll back-off (ns) of the roles that are not on the tensor core's critical path.  The epilogue groups
// spend most of their two-tile budget waiting for an accumulator: polled tightly, those waits were ~58 %
// of the SM's issued instructions (ncu source view), taking issue slots from the ReLU and UMMA warps.
#ifndef CNRX_WS_SLEEP_NS
#define CNRX_WS_SLEEP_NS 128
#endif
__device__ __forceinline__ void ws_wait_relaxed(uint64_t* bar, uint32_t parity) {
  if (CNRX_WS_SLEEP_NS > 0)
    mbar_wait_backoff<CNRX_WS_SLEEP_NS>(bar, parity);
  else
    mbar_wait(bar, parity);
}

// In-place ReLU of 16-byte chunks [lo, hi) of a shared-memory window, one warp, batches of 16 chunks per
// lane so all loads are in flight before the first store (shared-memory latency is long while the
// tensor core streams the other stages).
template <bool F16>
__device__ __forceinline__ void relu_chunks(uint32_t win, int lo, int hi, int lane) {
  for (int c0 = lo; c0 < hi; c0 += 32 * 16) {
    uint4 v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < hi) v[u] = lds128(win + static_cast<uint32_t>(c) * 16u);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = c0 + u * 32 + lane;
      v[u].x = relu2<F16>(v[u].x);
      v[u].y = relu2<F16>(v[u].y);
      v[u].z = relu2<F16>(v[u].z);
      v[u].w = relu2<F16>(v[u].w);
      if (c < hi) sts128(win + static_cast<uint32_t>(c) * 16u, v[u]);
    }
  }
}

template <int FL, bool F16>
__global__ void __launch_bounds__(kWsThreads, 1) conv_ws64_kernel(const __grid_constant__ WsLaunch L) {
  constexpr uint32_t IDESC = idesc_e16_f32<F16>(128, kN);
  constexpr bool kHead = FL > 0 && (FL & kWsHead) != 0;
  constexpr int kNS = kHead ? (FL >> 6) & 3 : 1;  // fused head: subnetworks (fold operands, cluster size)
  // fused head with the fold shape compiled in (bit 16): bits 8-9 step 1/2 is a product, 10-12 step
  // 0-2 has a ReLU, 13-15 step 0-2 has a BN; otherwise the fold is read from the launch (branch-free)
  constexpr bool kFoldSpec = kHead && (FL & (1 << 16)) != 0;
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_align1024(smem_dyn);
  const WsLayout lay = ws_layout(L.stages, L.win_alloc, kHead);
  float* s_bias = reinterpret_cast<float*>(smem + lay.par_off);
  float* s_s2 = s_bias + kC;
  float* s_t2 = s_s2 + kC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* full = bars;                  // [stages]
  uint64_t* empty = full + L.stages;      // [stages]
  uint64_t* tfull = empty + L.stages;     // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint64_t* rfull = tempty + 2;           // [2 groups][2 buffers] residual tile landed
  uint64_t* ready = rfull + 4;            // [stages] window ReLU'd in place (relu_in only)
  uint64_t* land = ready + L.stages;      // [2] (head) the other ranks' rows of the group's tile landed
  uint64_t* cons = land + 2;              // [2] (head) the other ranks have folded the group's tile
  uint64_t* hfull = cons + 2;             // [2 groups][2] (head) head UMMAs of group tile n (n & 1) done
  uint64_t* zready = hfull + 4;           // [2] (head) z rows of the group's current tile staged
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(zready + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int G = L.ngroups;
  const int g = blockIdx.x % G;
  const int local = blockIdx.x / G;
  const int nct = (static_cast<int>(gridDim.x) - g + G - 1) / G;
  const WsGroup& grp = L.g[g];
  const int64_t n_tiles = L.n_tiles;
  const bool has_res = FL < 0 ? grp.res_map_valid != 0 : (FL & kWsRes) != 0;
  const bool has_out2 = FL < 0 ? grp.out2_map_valid != 0 : (FL & kWsOut2) != 0;
  const bool relu_main = FL < 0 ? grp.relu != 0 : (FL & kWsRelu) != 0;
  const bool relu_in = FL < 0 ? grp.relu_in != 0 : (FL & kWsReluIn) != 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&ready[s], 1);  // input ReLU done (warp 18)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
      mbar_init(&rfull[2 * a], 1);
      mbar_init(&rfull[2 * a + 1], 1);
      if (kHead) {
        mbar_init(&land[a], kNS > 1 ? static_cast<uint32_t>(kNS - 1) : 1u);
        mbar_init(&cons[a], kNS > 1 ? static_cast<uint32_t>(kNS - 1) : 1u);
        mbar_init(&hfull[2 * a], 1);
        mbar_init(&hfull[2 * a + 1], 1);
        mbar_init(&zready[a], 8);
      }
    }
    fence_barrier_init();
  }
  if (kHead && warp >= 2) {
    head_tc_pack_weights(smem + lay.hw_off, L.head.w, L.head.nb, threadIdx.x - 64, kWsThreads - 64);
    fence_proxy_async_smem();
    float* s_fold = reinterpret_cast<float*>(smem + lay.fold_off);
    for (int e = threadIdx.x - 64; e < 3 * kC; e += kWsThreads - 64) {
      const int k = e / kC, c = e % kC;
      const bool on = k < L.head.ns && L.head.aff_s[k] != nullptr;
      s_fold[(2 * k) * kC + c] = on ? L.head.aff_s[k][c] : 1.f;
      s_fold[(2 * k + 1) * kC + c] = on ? L.head.aff_t[k][c] : 0.f;
    }
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
  if (kHead) cl_sync();  // every CTA's barriers initialised before any remote arrive / copy
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp >= 2 && warp < 6) {
    // weights -> TMEM: block b = pair*4 + kstep occupies columns [8b, 8b+8); lane = packed row
    const int q = warp & 3;
    const uint32_t* src = grp.wimg + (static_cast<size_t>(q * 32 + lane) * 8);
    // one 32-byte load per lane (a warp reads 1 KB contiguous: full sectors); kWB blocks' loads in flight
    // before their TMEM stores -- one dependent load -> store round trip per block was ~3.5 us of
    // prologue per launch, most of a small batch's block kernel (B = 1: 19 us per launch, 6 us of MMAs)
    constexpr int kWB = 6;
    static_assert((kPairs * kKSteps) % kWB == 0, "weight blocks per batch");
#pragma unroll 1
    for (int b0 = 0; b0 < kPairs * kKSteps; b0 += kWB) {
      u32x8 w8[kWB];
#pragma unroll
      for (int i = 0; i < kWB; ++i) w8[i] = ldg256(src + static_cast<size_t>(b0 + i) * 128 * 8);
#pragma unroll
      for (int i = 0; i < kWB; ++i)
        tmem_st8(tbase + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>((b0 + i) * 8), w8[i].v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // everything above is independent of the previous kernel (PDL: it overlapped that kernel's tail)
  pdl_trigger();
  pdl_wait();

  // input ReLU of one window (relu_in), by warp 18
  const int relu_n = (kN + 1 + 2 * grp.halo) * (kRB / 16);  // only the rows the UMMAs read
  auto relu_stage = [&](int jr, int lo, int hi) {
    const int s = jr % L.stages;
    ws_wait_relaxed(&full[s], static_cast<uint32_t>(jr / L.stages) & 1u);
    if (!(L.debug & 2)) relu_chunks<F16>(smem_u32(smem + lay.win_off + s * lay.win_stage), lo, hi, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&ready[s]);
  };

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) prefetch_tmap(&grp.in_map);
    const int nboxes = (kN + 1 + 2 * grp.halo + kBox - 1) / kBox;
    const uint32_t stage_tx = static_cast<uint32_t>(nboxes * kBox * kRB);
    long long tr_prod = 0;
    int j = 0;
    for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
      if (lane == 0) {
        const int s = j % L.stages;
        const uint32_t k = static_cast<uint32_t>(j / L.stages);
        const int64_t p0 = tile * kTileRows;
        const long long tp0 = L.trace ? clock64() : 0;
        ws_wait_relaxed(&empty[s], (k & 1u) ^ 1u);
        if (L.trace) tr_prod += clock64() - tp0;
        mbar_arrive_expect_tx(&full[s], stage_tx);
        uint8_t* win = smem + lay.win_off + s * lay.win_stage;
        const int32_t r0 = static_cast<int32_t>(p0 - grp.halo);
        for (int bx = 0; bx < nboxes; ++bx)
          tma_load_2d(win + bx * kBox * kRB, &grp.in_map, &full[s], 0, r0 + bx * kBox);
      }
    }
    if (L.trace && lane == 0) atomicAdd(&L.trace[kTraceProdWaitEmpty], static_cast<unsigned long long>(tr_prod));
  } else if (warp == 1 || warp == 19) {
    // ------------------------------ MMA issuers --------------------------------
    // Two issuing warps, one per accumulator stage (alternate tiles): the UMMA queue is shallow, so a
    // single issuer's per-tile barrier waits, commits and loop overhead leave the tensor pipe idle;
    // with two, one warp's tile keeps the pipe fed while the other does its bookkeeping.  Each warp's
    // tcgen05.commit tracks only its own UMMAs.
    // pair p: A-half tap (dt = -1 or +1, df), B-half tap dt + 1 (real for the first three pairs)
    const int me = warp == 1 ? 0 : 1;
    int32_t shift[kPairs];
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
      const int df = p % 3 - 1;
      const int dt = p < 3 ? -1 : 1;
      shift[p] = grp.halo + dt + df * grp.dil * L.geo.T1;
    }
    long long tr_full = 0, tr_tmem = 0, tr_issue = 0, tr_loop = 0, tr_commit = 0;
    const long long t_start = clock64();
    const unsigned long long g_start = globaltimer_ns();
    long long t_prev_end = t_start;
    int j = me;
    for (int64_t tile = local + static_cast<int64_t>(me) * nct; tile < n_tiles; tile += 2 * static_cast<int64_t>(nct), j += 2) {
      const int s = j % L.stages;
      const int a = j & 1;
      const long long tm0 = clock64();
      tr_loop += tm0 - t_prev_end;
      mbar_wait(relu_in ? &ready[s] : &full[s], static_cast<uint32_t>(j / L.stages) & 1u);
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
            umma_f16_ts(d_tmem, tbase + static_cast<uint32_t>((p * kKSteps + kk) * 8), bd, IDESC,
                         (p | kk) != 0 ? 1u : 0u);
          }
        }
        const long long tc0 = clock64();
        umma_commit(&empty[s]);
        umma_commit(&tfull[a]);
        tr_commit += clock64() - tc0;
      }
      __syncwarp();
      t_prev_end = clock64();
      tr_issue += t_prev_end - tm2;
    }
    if (L.trace && lane == 0 && me == 0) {  // per-tile figures of stage 0's issuer (half the tiles)
      j >>= 1;
      atomicAdd(&L.trace[kTraceTotal], static_cast<unsigned long long>(clock64() - t_start));
      trace_cta_window(L.trace, g_start);
      atomicAdd(&L.trace[kTraceMmaWaitFull], static_cast<unsigned long long>(tr_full));
      atomicAdd(&L.trace[kTraceMmaWaitTmem], static_cast<unsigned long long>(tr_tmem));
      atomicAdd(&L.trace[kTraceMmaIssue], static_cast<unsigned long long>(tr_issue));
      atomicAdd(&L.trace[kTraceTiles], static_cast<unsigned long long>(j));
      atomicAdd(&L.trace[kWsTraceLoop], static_cast<unsigned long long>(tr_loop));
      atomicAdd(&L.trace[kWsTraceCommit], static_cast<unsigned long long>(tr_commit));
    }
  } else if (warp == 18 && kHead) {
    // ------------------------------ fused head: head UMMA issuer ---------------
    // A warp of its own: a tcgen05.ld from a warp with UMMAs in flight waits for them, and the head
    // UMMAs queue behind the conv UMMAs in the tensor pipe.
    {
      const uint32_t hw_a = smem_u32(smem + lay.hw_off);
      int j = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) {
        const int e = j & 1;
        const uint32_t gn = static_cast<uint32_t>(j) >> 1;
        ws_wait_relaxed(&zready[e], gn & 1u);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t hb = 2u * static_cast<uint32_t>(e) + (gn & 1u);
          if (!(L.debug & 32)) head_tc_umma(tbase + kHeadCol + 16u * hb, smem_u32(smem + lay.stg_off + e * 2 * 128 * kRB), hw_a);
          umma_commit(&hfull[hb]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 18) {
    // ------------------------------ input ReLU (relu_in) ----------------------
    // The window is the B operand of the tensor core (async proxy): ReLU it in place with generic
    // 16-byte shared accesses, then fence the generic writes to the async proxy before the MMA warp
    // may read them.
    if (relu_in) {
      int j = 0;
      for (int64_t tile = local; tile < n_tiles; tile += nct, ++j) relu_stage(j, 0, relu_n);
    }
  } else {
    // ------------------------------ epilogue (warps 2..17) --------------------
    // Two groups of eight warps, group e owning accumulator stage e (tiles j with j % 2 == e), so one
    // group's TMEM reads overlap the other group's shared-memory writes and TMA stores.  In a group,
    // warp (q, H) covers TMEM lane quadrant q and accumulator columns [64H, 64H + 64) as two 32-column
    // chunks.
    const int e = (warp - 2) >> 3;     // epilogue group == accumulator stage
    const int q = warp & 3;            // TMEM lane quadrant: channels 16q .. 16q+15 (two 16-lane blocks)
    const int H = ((warp - 2) >> 2) & 1;
    const int t0 = lane & 3;           // column pair within an 8-column group
    const int ci = lane >> 2;          // channel within a 16-lane block
    const PlaneGeom geo = L.geo;
    uint8_t* stg = smem + lay.stg_off + e * 2 * 128 * kRB;
    const uint32_t stg_a = smem_u32(stg);
    float bias[2], s2v[2], t2v[2];
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) {
      const int ch = 16 * q + 8 * blk + ci;
      bias[blk] = s_bias[ch];
      s2v[blk] = s_s2[ch];
      t2v[blk] = s_t2[ch];
    }
    // Fused head (kHead): every rank stages its output tile (as for a TMA store), copies the rows
    // [hr0(d), hr1(d)) of it into rank d's receive slots (distributed shared memory), and folds its OWN
    // row range of all kNS tiles: fold pass -> z (bf16, in place of its own rows) -> head UMMAs (warp
    // 18) -> LLRs, read back at the group's next tile.  Symmetric, so every rank does a third of the fold.
    const float* s_fold = reinterpret_cast<const float*>(smem + lay.fold_off);
    constexpr int kHRows = kNS == 3 ? 48 : kNS == 2 ? 64 : 128;  // fold rows per rank (multiple of 8)
    const int hr0 = g * kHRows, hr1 = hr0 + kHRows < 128 ? hr0 + kHRows : 128;
    const int gtid = ((warp - 2) & 7) * 32 + lane;  // thread in the epilogue group
    const bool relu2_only = FL < 0 ? grp.s2 == nullptr : (FL & kWsOut2Bn) == 0;
    const bool lead = ((warp - 2) & 7) == 0 && lane == 0;
    // ldmatrix / stmatrix row addresses: thread a -> matrix a/8 (8-row group), row a%8
    const int arow = ((lane >> 3) << 3) + (lane & 7);
    long long tr_ew = 0, tr_comb = 0, tr_sw = 0, tr_wr = 0;
    // The group's lead thread streams its own residual tiles through two buffers: the load for the
    // group's tile k+2 is issued once every warp of the group has read tile k's, two group tiles
    // (four tile periods) ahead of its use.
    uint8_t* rbuf0 = smem + lay.res_off + e * 2 * 128 * kRB;
    auto load_res = [&](int64_t t, int b) {
      uint8_t* dst = rbuf0 + b * 128 * kRB;
      mbar_arrive_expect_tx(&rfull[2 * e + b], 128u * kRB);
      for (int bx = 0; bx < 4; ++bx)
        tma_load_2d(dst + bx * kBox * kRB, &grp.res_map, &rfull[2 * e + b], 0, static_cast<int32_t>(t * kTileRows + bx * kBox));
    };
    const int64_t gstride = 2 * static_cast<int64_t>(nct);
    // head results of group tile m (TMEM lane = tile row) -> LLRs of this rank's rows
    auto head_drain = [&](uint32_t m, int64_t mtile) {
      const uint32_t hb = 2u * static_cast<uint32_t>(e) + (m & 1u);
      if (H == 0) {
        ws_wait_relaxed(&hfull[hb], (m >> 1) & 1u);
        tc_fence_after();
        uint32_t d[8];
        tmem_ld8(tbase + kHeadCol + 16u * hb + (static_cast<uint32_t>(q * 32) << 16), d);
        tmem_ld_wait();
        tc_fence_before();
        const int row = q * 32 + lane;
        const int64_t pr = mtile * kTileRows + row;
        if (row >= hr0 && row < hr1 && row < kTileRows && geo.valid(pr)) {
          int b, t, f;
          geo.coords(pr, b, t, f);
          const int nb = L.head.nb;
          float* dst = L.head.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * nb;
          if (nb == 4) {
            *reinterpret_cast<float4*>(dst) =
                make_float4(__uint_as_float(d[0]) + L.head.b[0], __uint_as_float(d[1]) + L.head.b[1],
                            __uint_as_float(d[2]) + L.head.b[2], __uint_as_float(d[3]) + L.head.b[3]);
          } else {
            for (int k = 0; k < nb; ++k) dst[k] = __uint_as_float(d[k]) + L.head.b[k];
          }
        }
      }
    };
    // fold of this rank's rows: head.cu's fold (fp32, fold order = cluster rank) over 16-byte chunks
    // (8 channels of a row, as 4 packed channel pairs), z written over the own tile's rows
    auto fold_pass = [&]() {
      const int nch = (hr1 - hr0) * 8;
      for (int c = gtid; c < nch; c += 256) {
        const int row = hr0 + (c >> 3), c8 = c & 7;
        const uint32_t off = sw128(static_cast<uint32_t>(row), static_cast<uint32_t>(c8 * 16));
        uint4 v[kNS];
#pragma unroll
        for (int k = 0; k < kNS; ++k) {
          const int slot = k < g ? k : k - 1;  // receive slot of rank k's rows
          v[k] = lds128(k == g ? stg_a + off
                               : stg_a + sw128(static_cast<uint32_t>(128 + slot * kHRows + row - hr0), static_cast<uint32_t>(c8 * 16)));
        }
        uint32_t zo[4];
#pragma unroll
        for (int pp = 0; pp < 4; ++pp) {
          const int ch = 8 * c8 + 2 * pp;
          auto word = [&](int k) {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(&v[k]);
            return unpack2<F16>(w[pp]);
          };
          float2 z = word(0);
          auto post = [&](auto kc) {
            constexpr int k = decltype(kc)::value;
            if (kFoldSpec ? ((FL >> (13 + k)) & 1) != 0 : L.head.aff_s[k] != nullptr) {
              const float2 sv = *reinterpret_cast<const float2*>(s_fold + (2 * k) * kC + ch);
              const float2 tv = *reinterpret_cast<const float2*>(s_fold + (2 * k + 1) * kC + ch);
              z = __ffma2_rn(z, sv, tv);
            }
            if (kFoldSpec ? ((FL >> (10 + k)) & 1) != 0 : L.head.relu[k] != 0) {
              z.x = fmaxf(z.x, 0.f);
              z.y = fmaxf(z.y, 0.f);
            }
          };
          auto step = [&](auto kc) {
            constexpr int k = decltype(kc)::value;
            const float2 zk = word(k);
            const bool mul = kFoldSpec ? ((FL >> (7 + k)) & 1) != 0 : L.head.op[k] == PW_MUL;
            z = mul ? __fmul2_rn(z, zk) : __fadd2_rn(z, zk);
            post(kc);
          };
          post(std::integral_constant<int, 0>{});
          if constexpr (kNS > 1) step(std::integral_constant<int, 1>{});
          if constexpr (kNS > 2) step(std::integral_constant<int, 2>{});
          zo[pp] = pack2<F16>(z.x, z.y);
        }
        sts128(stg_a + off, make_uint4(zo[0], zo[1], zo[2], zo[3]));
      }
    };
    if (has_res && lead) {
      prefetch_tmap(&grp.res_map);
      const int64_t t0_ = local + static_cast<int64_t>(e) * nct;
      if (t0_ < n_tiles) load_res(t0_, 0);
      if (t0_ + gstride < n_tiles) load_res(t0_ + gstride, 1);
    }
    int j = e;
    for (int64_t tile = local + static_cast<int64_t>(e) * nct; tile < n_tiles; tile += 2 * static_cast<int64_t>(nct), j += 2) {
      const int64_t p0 = tile * kTileRows;
      const long long te0 = clock64();
      ws_wait_relaxed(&tfull[e], static_cast<uint32_t>(j >> 1) & 1u);
      const long long te1 = clock64();
      tr_ew += te1 - te0;
      const uint32_t gn = static_cast<uint32_t>(j) >> 1;  // this group's tile count
      // staging buffer free?  TMA store: this group's previous store has read it.  Fused head: every
      // other rank has folded the previous tile (so the copies out of it, and into their receive slots,
      // are complete), and this rank's head UMMAs have read its z rows (head_drain).
      if (lead) {
        if (kHead) {
          if (kNS > 1 && gn >= 1 && !(L.debug & 128)) cl_wait(&cons[e], (gn - 1) & 1u);
        } else {
          bulk_wait_read0();
        }
      }
      if (kHead && gn >= 1) head_drain(gn - 1, tile - gstride);
      epi_group_sync(e);
      const int kb = (j >> 1) & 1;  // residual buffer of this group tile
      if (has_res) ws_wait_relaxed(&rfull[2 * e + kb], static_cast<uint32_t>(j >> 2) & 1u);
      const uint32_t rbuf_a = smem_u32(rbuf0 + kb * 128 * kRB);
      const long long te2 = clock64();
      tr_sw += te2 - te1;
      tc_fence_after();
      // Chunk h = accumulator columns c = 64H + 32h + [0, 32).  Lanes 16k + i / 16k + 8 + i hold the
      // A / B tap partial sums of channel 8k + i, so output row c = A[c] + B[c+1] needs one shuffle
      // for odd c (B[c+1] sits with the neighbouring column pair) and none for even c.
      // validity of this warp's 64 rows (padding rows are stored as zeros): one bit per row
      uint32_t vmask[2];
#pragma unroll
      for (int w = 0; w < 2; ++w) vmask[w] = __ballot_sync(0xffffffffu, geo.valid(p0 + 64 * H + 32 * w + lane));
      const uint32_t tq = tbase + kAcc0 + static_cast<uint32_t>(e * kN + 64 * H) + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t a0[16], a1[16], xb;
        tmem_ld16x256b_x4(tq + 32 * h, a0);
        tmem_ld16x256b_x4(tq + (16u << 16) + 32 * h, a1);
        if (H == 0 || h == 0) {
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(xb) : "r"(tq + 32 * h + 32) : "memory");
        } else {
          xb = 0;  // column 128 would only feed row 127, which is never stored
        }
        tmem_ld_wait();
        if (h == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_relaxed(&tempty[e]);
        }
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          uint32_t (&a)[16] = blk == 0 ? a0 : a1;
          uint32_t rres[4] = {0u, 0u, 0u, 0u};
          if (has_res) {
            // residual rows 64H + 32h + 8i + arow%8 (matrix i), channel chunk 2q + blk
            const uint32_t row = static_cast<uint32_t>(64 * H + 32 * h + arow);
            ldsm_x4_trans(rbuf_a + sw128(row, static_cast<uint32_t>((2 * q + blk) * 16)), rres);
          }
          const float bnd = __uint_as_float(__shfl_sync(0xffffffffu, xb, 16 * blk + 8 + ci));
          uint32_t o[4], o2[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t snd = t0 == 0 ? (i < 3 ? a[4 * (i + 1) + 2] : 0u) : a[4 * i + 2];
            float got = __uint_as_float(__shfl_sync(0xffffffffu, snd, t0 == 3 ? lane - 3 : lane + 1));
            if (i == 3 && t0 == 3) got = bnd;
            float y0 = __uint_as_float(a[4 * i + 0]) + __uint_as_float(a[4 * i + 3]) + bias[blk];
            float y1 = __uint_as_float(a[4 * i + 1]) + got + bias[blk];
            if (has_res) {
              const float2 rf = unpack2<F16>(rres[i]);
              y0 += rf.x;
              y1 += rf.y;
            }
            if (relu_main) {
              y0 = fmaxf(y0, 0.f);
              y1 = fmaxf(y1, 0.f);
            }
            const int rb = 8 * i + 2 * t0;  // row 64H + 32h + rb
            const bool v0 = (vmask[h] >> rb) & 1u, v1 = (vmask[h] >> (rb + 1)) & 1u;
            if (!v0) y0 = 0.f;
            if (!v1) y1 = 0.f;
            o[i] = pack2<F16>(y0, y1);
            if (has_out2) {
              if (relu2_only) {
                o2[i] = relu2<F16>(o[i]);
              } else {
                const float2 f = unpack2<F16>(o[i]);
                const float x0 = fmaxf(f.x * s2v[blk] + t2v[blk], 0.f);
                const float x1 = fmaxf(f.y * s2v[blk] + t2v[blk], 0.f);
                o2[i] = pack2<F16>(v0 ? x0 : 0.f, v1 ? x1 : 0.f);
              }
            }
          }
          const uint32_t row = static_cast<uint32_t>(64 * H + 32 * h + arow);
          const uint32_t off = sw128(row, static_cast<uint32_t>((2 * q + blk) * 16));
          if (!(L.debug & 1)) {
            stsm_x4_trans(stg_a + off, o);
            if (has_out2) stsm_x4_trans(stg_a + 128 * kRB + off, o2);
          }
        }
      }
      const long long te3 = clock64();
      tr_comb += te3 - te2;
      fence_proxy_async_smem();
      epi_group_sync(e);
      if (kHead) {
        if (lead) {
          // rows of rank d -> rank d's receive slot for this rank
#pragma unroll
          for (int d = 0; d < kNS; ++d) {
            if (d == g || (L.debug & 128)) continue;
            const int d0 = d * kHRows, dn = (d0 + kHRows < 128 ? d0 + kHRows : 128) - d0;
            const int slot = g < d ? g : g - 1;
            const uint32_t zb = cl_map(&land[e], static_cast<uint32_t>(d));
            cl_arrive_expect_tx(zb, static_cast<uint32_t>(dn) * kRB);
            bulk_copy_to_cta(cl_map(stg + (128 + slot * kHRows) * kRB, static_cast<uint32_t>(d)), stg + d0 * kRB,
                             static_cast<uint32_t>(dn) * kRB, zb);
          }
          if (has_res && tile + 2 * gstride < n_tiles) load_res(tile + 2 * gstride, kb);
        }
        if (kNS > 1 && !(L.debug & 128)) cl_wait(&land[e], gn & 1u);  // the other ranks' rows of this tile
        if (!(L.debug & 64)) fold_pass();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&zready[e]);  // warp 18: head UMMAs over the z rows
        epi_group_sync(e);
        if (lead && !(L.debug & 128))  // receive slots read: the senders may reuse them (and their staging)
          for (int r = 0; r < kNS; ++r)
            if (r != g) cl_arrive(cl_map(&cons[e], static_cast<uint32_t>(r)));
      } else if (lead && !(L.debug & 1)) {
        tma_store_2d(&grp.out_map, stg, 0, static_cast<int32_t>(p0));
        if (has_out2) tma_store_2d(&grp.out2_map, stg + 128 * kRB, 0, static_cast<int32_t>(p0));
        bulk_commit();
        if (has_res && tile + 2 * gstride < n_tiles) load_res(tile + 2 * gstride, kb);
      }
      tr_wr += clock64() - te3;
    }
    if (kHead && j > e)
      head_drain((static_cast<uint32_t>(j) >> 1) - 1,
                 local + static_cast<int64_t>(e) * nct + (static_cast<int64_t>(j >> 1) - 1) * gstride);
    if (lead) bulk_wait0();
    if (L.trace && lead && e == 0 && (!kHead || g == ((L.debug & 16) ? 1 : 0))) {  // (fused head: rank 0, or rank 1 with debug bit 4)
      atomicAdd(&L.trace[kTraceEpiWaitFull], static_cast<unsigned long long>(tr_ew));
      atomicAdd(&L.trace[kWsTraceCombine], static_cast<unsigned long long>(tr_comb));
      atomicAdd(&L.trace[kWsTraceStageWait], static_cast<unsigned long long>(tr_sw));
      atomicAdd(&L.trace[kWsTraceWrite], static_cast<unsigned long long>(tr_wr));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (kHead) cl_sync();  // no CTA leaves while a peer may still signal its barriers or copy into it
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

void conv_ws64_pack_weights(const float* w, const float* scale, bool fp16, uint32_t* img) {
  // w: reference layout [3][3][64][64] = [dt+1][df+1][ci][co]; img: [block = pair*4 + kstep][lane][8 u32]
  std::memset(img, 0, conv_ws64_wimg_bytes());
  for (int p = 0; p < kPairs; ++p) {
    const int df = p % 3 - 1;
    const int dtA = p < 3 ? -1 : 1;
    for (int half = 0; half < 2; ++half) {
      const int dt = dtA + half;
      const bool real = half == 0 || p < 3;
      for (int co = 0; co < kC; ++co) {
        const int lane = 16 * (co / 8) + 8 * half + co % 8;
        for (int ci = 0; ci < kC; ++ci) {
          float v = 0.f;
          if (real) {
            v = w[((static_cast<size_t>(dt + 1) * 3 + (df + 1)) * kC + ci) * kC + co];
            if (scale) v *= scale[co];
          }
          const uint16_t bits = e16_from_float_host(v, fp16);
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

namespace {

int group_flags(const WsGroup& g) {
  return (g.res_map_valid ? kWsRes : 0) | (g.out2_map_valid ? kWsOut2 : 0) | (g.s2 ? kWsOut2Bn : 0) |
         (g.relu ? kWsRelu : 0) | (g.relu_in ? kWsReluIn : 0);
}

template <int FL, bool F16>
void launch_flh(const WsLaunch& L, const WsLayout& lay, int grid, cudaStream_t stream) {
  ensure_smem_attr(reinterpret_cast<const void*>(conv_ws64_kernel<FL, F16>), static_cast<int>(lay.total));
  launch_pdl(conv_ws64_kernel<FL, F16>, dim3(grid), dim3(kWsThreads), lay.total, stream, L);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {  // (launch_pdl throws on launch errors; this catches sticky ones)
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, conv_ws64_kernel<FL, F16>);
    throw Error(4, std::string("conv_ws64 launch failed: ") + cudaGetErrorString(err) + " (regs " +
                       std::to_string(fa.numRegs) + ", max threads " + std::to_string(fa.maxThreadsPerBlock) +
                       ", static smem " + std::to_string(fa.sharedSizeBytes) + ", dynamic " +
                       std::to_string(lay.total) + ")");
  }
}

template <int FL>
void launch_fl(const WsLaunch& L, const WsLayout& lay, int grid, cudaStream_t stream) {
  if (L.fp16)
    launch_flh<FL, true>(L, lay, grid, stream);
  else
    launch_flh<FL, false>(L, lay, grid, stream);
}

// Fused-head launches (bf16 plans only): clusters of ngroups CTAs (one per subnetwork), as many as can
// be co-resident.
template <int FL>
void launch_head(const WsLaunch& L, const WsLayout& lay, cudaStream_t stream) {
  auto kern = conv_ws64_kernel<FL, false>;
  ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(lay.total));
  static const bool no_pdl = std::getenv("CNRX_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kWsThreads);
  cfg.dynamicSmemBytes = lay.total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(L.ngroups);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // co-resident clusters, per (device, cluster size)
  static int cache[64][5] = {};
  int dev = 0;
  CNRX_CUDA(cudaGetDevice(&dev));
  int& ncl = cache[dev & 63][L.ngroups];
  if (ncl == 0) {
    cfg.gridDim = dim3(static_cast<unsigned>(L.ngroups * 148));
    CNRX_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
    if (ncl <= 0) throw Error(4, "fused-head conv: no cluster of " + std::to_string(L.ngroups) + " CTAs fits an SM set");
    if (std::getenv("CNRX_TRACE")) fprintf(stderr, "[trace] fused-head conv: %d co-resident clusters of %d\n", ncl, L.ngroups);
  }
  const int64_t nc = L.n_tiles < ncl ? L.n_tiles : ncl;
  cfg.gridDim = dim3(static_cast<unsigned>(nc * L.ngroups));
  cfg.numAttrs = 2;
  CNRX_CUDA(cudaLaunchKernelEx(&cfg, kern, L));
}

}  // namespace

size_t conv_ws64_head_smem_bytes(int stages, int win_alloc) { return ws_layout(stages, win_alloc, true).total; }

const char* conv_ws64_launch(const WsLaunch& L, int num_sms, cudaStream_t stream) {
  if (L.head_on) {
    if (L.fp16) throw Error(4, "internal: the fused-head conv is bf16-only");
    const WsLayout lay = ws_layout(L.stages, L.win_alloc, true);
    for (int i = 0; i < L.ngroups; ++i)
      if (group_flags(L.g[i]) != kWsRes) throw Error(4, "internal: fused-head conv needs residual-only epilogues");
    if (L.ngroups != L.head.ns || L.head.ns > 3 || L.head.nb > 8) throw Error(4, "internal: fused-head shape");
    const WsHead& h = L.head;
    const bool cfg2_fold = h.ns == 3 && h.op[1] == PW_MUL && h.op[2] == PW_MUL && !h.aff_s[0] && h.aff_s[1] &&
                           h.aff_s[2] && !h.relu[0] && !h.relu[1] && !h.relu[2];
    if (cfg2_fold) {  // build_conet's mul -> BN -> mul -> BN tail (CoNet-ResNet)
      launch_head<kWsRes | kWsHead | (3 << 6) | (3 << 8) | (6 << 13) | (1 << 16)>(L, lay, stream);
      return "conv_ws64_kernel<head>";
    }
    switch (L.head.ns) {
      case 1: launch_head<kWsRes | kWsHead | (1 << 6)>(L, lay, stream); break;
      case 2: launch_head<kWsRes | kWsHead | (2 << 6)>(L, lay, stream); break;
      default: launch_head<kWsRes | kWsHead | (3 << 6)>(L, lay, stream); break;
    }
    return "conv_ws64_kernel<head>";
  }
  const WsLayout lay = ws_layout(L.stages, L.win_alloc);
  const int64_t work = static_cast<int64_t>(L.ngroups) * L.n_tiles;
  int grid = static_cast<int>(work < num_sms ? work : num_sms);
  if (grid < L.ngroups) grid = L.ngroups;
  int fl = group_flags(L.g[0]);
  for (int i = 1; i < L.ngroups; ++i)
    if (group_flags(L.g[i]) != fl) fl = kWsDynamic;
  switch (fl) {
    case kWsRelu: launch_fl<kWsRelu>(L, lay, grid, stream); break;                         // block conv 1
    case kWsRelu | kWsReluIn: launch_fl<kWsRelu | kWsReluIn>(L, lay, grid, stream); break; // conv 1, ReLU on load
    case kWsRes | kWsOut2: launch_fl<kWsRes | kWsOut2>(L, lay, grid, stream); break;       // block conv 2
    case kWsRes: launch_fl<kWsRes>(L, lay, grid, stream); break;                           // last block conv 2
    case kWsRes | kWsOut2 | kWsOut2Bn: launch_fl<kWsRes | kWsOut2 | kWsOut2Bn>(L, lay, grid, stream); break;
    case 0: launch_fl<0>(L, lay, grid, stream); break;
    default: launch_fl<kWsDynamic>(L, lay, grid, stream); break;
  }
  return L.fp16 ? "conv_ws64_kernel<f16>" : "conv_ws64_kernel";
}

}  // namespace cnrx
