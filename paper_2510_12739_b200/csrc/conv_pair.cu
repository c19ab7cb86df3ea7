// conv_pair.cu — the 96 -> 96 channel 3x3 convolution (cfg3 / cfg4 subnetworks) on CTA PAIRS:
// tcgen05.mma.cta_group::2 with M = 256 plane rows, N = 96 output channels.
//
// Same math and epilogue as conv_tc.cu's <96,96,3> instantiation (replaces conetrx::conv2d,
// kernels.hpp:47-91, with the fused BN / ReLU / residual / pre-activation epilogue; see conv_tc.cu).
// Why pairs: the single-CTA SS UMMA 128 x 96 x 16 reads 4 KB (A) + 3 KB (B) of shared memory per
// 48-cycle instruction = 149 B/clk, above the SM's ~128 B/clk, so that kernel is shared-memory bound
// before its epilogue and TMA traffic are even counted.  In a pair each SM supplies its own 128 window
// rows (A) and HALF of the weights (B: output channels 48r .. 48r+47), so an instruction reads 5.5 KB
// per SM and each SM keeps only half the weight image resident (83 KB).  The accumulator for each
// CTA's own 128 rows x all 96 channels lands in that CTA's TMEM (pinned by tools/probes/pair_probe.cu),
// so the epilogue is the single-CTA one, unchanged.
//
// Protocol (leader = cluster rank 0 issues every UMMA):
//   * both producers TMA their own window stage; the leader's full[s] barrier expects both CTAs' bytes
//     (the peer loads with the .cta_group::2 TMA form, signalling the leader's barrier);
//   * UMMA completion is multicast-committed to both CTAs' empty[s] (window free) and tfull[a];
//   * both CTAs' epilogue warps arrive on the leader's tempty[a] (count 16) after draining TMEM;
//   * weights: each CTA bulk-loads its half; the peer reports completion on the leader's wpeer barrier;
//   * TMEM is allocated / freed with cta_group::2 (same column base in both CTAs).
// Warp roles per CTA (320 threads): warp 0 producer, warp 1 TMEM allocator + (leader) UMMA issuer,
// warps 2-9 epilogue (two per TMEM lane quadrant).  Tiles: pair-tile k covers 128-row tiles 2k (rank 0) and 2k + 1 (rank 1).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "conv_pair.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kC = 96;               // channels in and out
constexpr int kHalfN = 48;           // output channels per CTA (B rows)
constexpr int kRB0 = 128, kRB1 = 64; // bytes per row of K-chunk 0 (64 ch) / chunk 1 (32 ch)
constexpr int kTapBytes = kHalfN * (kRB0 + kRB1);  // 9216: one tap of this CTA's weight half
constexpr int kWBytes = 9 * kTapBytes;             // 82944
constexpr int kTmemCols = 256;       // 2 accumulator stages x 96 columns
constexpr int kBox = 32;
constexpr int kThreads = 416;   // producer, UMMA, 8 epilogue warps, store warp, 2 input-ReLU warps
constexpr int kStoreWarp = 10;
constexpr int kReluWarp0 = 11, kReluWarps = 2;
constexpr uint32_t kTileBytes = 128u * (kRB0 + kRB1);  // one 128-row tile of a 96-ch plane (24 KB)

// `staged` (launches with a residual and/or a second output): residual tiles arrive by TMA into rbuf,
// the epilogue writes y over them in place (same swizzled positions) and the pre-activated copy into
// o2buf, and the store warp writes both planes with TMA.  Those launches keep 2 window stages.
struct PairLayout {
  uint32_t w_off, win_off, win_stage, win_c1, rbuf_off, o2_off, par_off, bar_off, total;
};
__host__ __device__ inline PairLayout pair_layout(int stages, int win_alloc, bool staged) {
  PairLayout s{};
  s.w_off = 0;
  s.win_off = (kWBytes + 1023u) & ~1023u;
  s.win_c1 = (static_cast<uint32_t>(win_alloc * kRB0) + 1023u) & ~1023u;
  s.win_stage = (s.win_c1 + static_cast<uint32_t>(win_alloc * kRB1) + 1023u) & ~1023u;
  uint32_t off = s.win_off + static_cast<uint32_t>(stages) * s.win_stage;
  s.rbuf_off = off;                  // staged: 2 x [128 rows: 64 ch SW128 | 32 ch SW64]
  if (staged) off += 2u * kTileBytes;
  s.o2_off = off;                    // staged: 1 x the same
  if (staged) off += kTileBytes;
  s.par_off = off;                   // bias, s2, t2
  off += 3u * kC * 4u;
  s.bar_off = (off + 15u) & ~15u;
  s.total = s.bar_off + 256 + 1024;
  return s;
}
// byte offset of channels [ch, ch+8) of tile row r in a staged tile buffer
__device__ __forceinline__ uint32_t tile_off(uint32_t r, uint32_t ch) {
  return ch < 64 ? r * 128u + ((((ch >> 3) ^ (r & 7u))) << 4)
                 : 128u * kRB0 + r * 64u + (((((ch - 64) >> 3) ^ ((r >> 1) & 3u))) << 4);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void* p, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(smem_u32(p)), "r"(rank));
  return d;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Arrival that orders nothing but itself: for "accumulator drained" signals, whose only precondition
// (the TMEM loads completed) is already established by tcgen05.wait::ld.  A release.cluster arrive
// would first wait for this warp's outstanding global stores to become cluster-visible.
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load into this CTA's shared memory, completion counted on the (leader's) barrier at cluster_bar
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const void* tmap, uint32_t cluster_bar, int32_t c0,
                                                int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(cluster_bar)
      : "memory");
}
__device__ __forceinline__ void umma_f16_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// completion of this thread's prior UMMAs arrives on the barrier at the same offset in both CTAs
__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(static_cast<uint16_t>(3))
               : "memory");
}

template <bool F16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    conv_pair96_kernel(const __grid_constant__ TcLaunch L) {
  constexpr uint32_t IDESC = idesc_e16_f32<F16>(256, kC);
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_align1024(smem_dyn);
  const bool staged = (L.flags & kPairStaged) != 0;
  const PairLayout lay = pair_layout(L.stages, L.win_alloc, staged);
  // tile buffer (residual in / y out) of pair-tile j and the parity of its use
  auto tbuf = [](int jj) { return jj & 1; };
  auto tpar = [](int jj) { return static_cast<uint32_t>(jj >> 1) & 1u; };
  uint8_t* sW = smem + lay.w_off;
  float* s_bias = reinterpret_cast<float*>(smem + lay.par_off);
  float* s_s2 = s_bias + kC;
  float* s_t2 = s_s2 + kC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* w_full = bars;             // own weight half landed
  uint64_t* wpeer = bars + 1;          // (leader) the peer's weight half landed
  uint64_t* full = bars + 2;           // [stages] (leader) both window halves landed
  uint64_t* empty = full + L.stages;   // [stages] window stage consumed (multicast commit)
  uint64_t* tfull = empty + L.stages;  // [2] accumulator ready (multicast commit)
  uint64_t* tempty = tfull + 2;        // [2] (leader) accumulator drained by both CTAs
  uint64_t* rfull = tempty + 2;        // [2] staged: residual tile landed
  uint64_t* rempty = rfull + 2;        // [2] staged: tile buffer's TMA store has read it
  uint64_t* sfull = rempty + 2;        // [2] staged: all epilogue warps wrote the tile buffer
  uint64_t* o2free = sfull + 2;        // staged: o2buf's TMA store has read it
  uint64_t* lfull = o2free + 1;        // [stages] (ReLU-on-load) this CTA's window stage landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lfull + L.stages);
  const bool relu_in = (L.flags & kPairReluIn) != 0;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int G = L.ngroups;
  const int pair = blockIdx.x >> 1;
  const int n_pairs = static_cast<int>(gridDim.x) >> 1;
  const int g = pair % G;
  const int local = pair / G;
  const int npc = (n_pairs - g + G - 1) / G;
  const TcGroup& grp = L.g[g];
  const int64_t n_tiles = L.geo.n_tiles;
  const int64_t n_ptiles = (n_tiles + 1) / 2;

  if (threadIdx.x == 0) {
    mbar_init(w_full, 1);
    mbar_init(wpeer, 1);
    for (int s = 0; s < L.stages; ++s) {
      // ReLU-on-load: the leader's full[s] completes when both CTAs' ReLU warps have processed their
      // window halves (2 x kReluWarps arrivals); otherwise on both CTAs' TMA bytes
      mbar_init(&full[s], relu_in ? 2 * kReluWarps : 1);
      mbar_init(&empty[s], 1);
      mbar_init(&lfull[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 16);  // 8 epilogue warps x 2 CTAs
      mbar_init(&rfull[a], 1);
      mbar_init(&rempty[a], 1);
      mbar_init(&sfull[a], 8);
    }
    mbar_init(o2free, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp >= 2 && warp < kStoreWarp) {
    for (int c = threadIdx.x - 64; c < kC; c += 256) {
      s_bias[c] = grp.bias[c];
      s_s2[c] = grp.s2 ? grp.s2[c] : 1.f;
      s_t2[c] = grp.t2 ? grp.t2[c] : 0.f;
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised before any remote arrive / TMA completion
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ------------------------------ TMA producer (both CTAs) ------------------
    if (lane == 0) {
      prefetch_tmap(&grp.map[0]);
      prefetch_tmap(&grp.map[1]);
      // this CTA's weight half: per tap, rows 48r .. 48r+47 of both K-chunk blocks of conv_tc's image
      mbar_arrive_expect_tx(w_full, kWBytes);
      const uint8_t* wimg = grp.wimg;
      for (int t = 0; t < 9; ++t) {
        const uint8_t* tap = wimg + static_cast<size_t>(t) * kC * kC * 2;
        bulk_load(sW + t * kTapBytes, tap + rank * kHalfN * kRB0, kHalfN * kRB0, w_full);
        bulk_load(sW + t * kTapBytes + kHalfN * kRB0, tap + kC * kRB0 + rank * kHalfN * kRB1, kHalfN * kRB1, w_full);
      }
      if (!leader) {
        mbar_wait(w_full, 0);
        mbar_arrive_cluster(map_to_rank(wpeer, 0));
      }
      const int nboxes = L.win_alloc / kBox;
      const uint32_t stage_tx = static_cast<uint32_t>(nboxes * kBox * (kRB0 + kRB1));
      int j = 0;
      for (int64_t k = local; k < n_ptiles; k += npc, ++j) {
        const int s = j % L.stages;
        mbar_wait(&empty[s], (static_cast<uint32_t>(j / L.stages) & 1u) ^ 1u);
        uint8_t* win = smem + lay.win_off + s * lay.win_stage;
        const int32_t r0 = static_cast<int32_t>((2 * k + rank) * 128 - grp.halo);
        if (relu_in) {  // own window on the own barrier; the ReLU warps report to the leader
          mbar_arrive_expect_tx(&lfull[s], stage_tx);
          for (int bx = 0; bx < nboxes; ++bx) {
            tma_load_2d(win + bx * kBox * kRB0, &grp.map[0], &lfull[s], 0, r0 + bx * kBox);
            tma_load_2d(win + lay.win_c1 + bx * kBox * kRB1, &grp.map[1], &lfull[s], 0, r0 + bx * kBox);
          }
        } else {
          const uint32_t fb = map_to_rank(&full[s], 0);
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * stage_tx);
          for (int bx = 0; bx < nboxes; ++bx) {
            tma_load_2d_2sm(win + bx * kBox * kRB0, &grp.map[0], fb, 0, r0 + bx * kBox);
            tma_load_2d_2sm(win + lay.win_c1 + bx * kBox * kRB1, &grp.map[1], fb, 0, r0 + bx * kBox);
          }
        }
        const int64_t tile = 2 * k + rank;
        if (staged && grp.res && tile < n_tiles) {
          const int b = tbuf(j);
          mbar_wait(&rempty[b], tpar(j) ^ 1u);
          mbar_arrive_expect_tx(&rfull[b], kTileBytes);
          uint8_t* rb = smem + lay.rbuf_off + b * kTileBytes;
          tma_load_2d(rb, &grp.pres[0], &rfull[b], 0, static_cast<int32_t>(tile * 128));
          tma_load_2d(rb + 128 * kRB0, &grp.pres[1], &rfull[b], 0, static_cast<int32_t>(tile * 128));
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ UMMA issuer (leader only) -----------------
    if (leader) {
      mbar_wait(w_full, 0);
      mbar_wait(wpeer, 0);
      tc_fence_after();
      const uint32_t sW_a = smem_u32(sW);
      const int32_t T1 = L.geo.T1;
      int j = 0;
      for (int64_t k = local; k < n_ptiles; k += npc, ++j) {
        const int s = j % L.stages;
        const int a = j & 1;
        if (relu_in)
          mbar_wait_cluster(&full[s], static_cast<uint32_t>(j / L.stages) & 1u);  // both CTAs' ReLU passes
        else
          mbar_wait(&full[s], static_cast<uint32_t>(j / L.stages) & 1u);
        mbar_wait(&tempty[a], (static_cast<uint32_t>(j >> 1) & 1u) ^ 1u);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t win = smem_u32(smem + lay.win_off + s * lay.win_stage);
          const uint32_t d_tmem = tbase + static_cast<uint32_t>(a * kC);
          uint32_t acc = 0;
#pragma unroll 1
          for (int tap = 0; tap < 9; ++tap) {
            const int dt = tap / 3 - 1, df = tap % 3 - 1;
            const int row = grp.halo + dt + df * grp.dil * T1;
            const uint32_t a0 = win + static_cast<uint32_t>(row * kRB0);
            const uint32_t a1 = win + lay.win_c1 + static_cast<uint32_t>(row * kRB1);
            const uint32_t b0 = sW_a + static_cast<uint32_t>(tap * kTapBytes);
            const uint32_t b1 = b0 + kHalfN * kRB0;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              umma_f16_2sm(d_tmem, make_sdesc(a0 + kk * 32, 8 * kRB0, kSwizzle128, 0),
                            make_sdesc(b0 + kk * 32, 8 * kRB0, kSwizzle128, 0), IDESC, acc);
              acc = 1;
            }
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
              umma_f16_2sm(d_tmem, make_sdesc(a1 + kk * 32, 8 * kRB1, kSwizzle64, 0),
                            make_sdesc(b1 + kk * 32, 8 * kRB1, kSwizzle64, 0), IDESC, 1);
          }
          umma_commit_2sm(&empty[s]);  // window stages of both CTAs free
          umma_commit_2sm(&tfull[a]);  // both CTAs' accumulators ready
        }
        __syncwarp();
      }
    }
  } else if (warp >= kReluWarp0) {
    // ------------------------------ input ReLU (ReLU-on-load launches) ---------
    // in place over this CTA's window stage (16-byte chunks of both K-chunk blocks; ReLU commutes with the
    // 16-bit rounding, so the values equal a pre-activated plane's), then a release arrive on the
    // leader's full[s]: its UMMAs read both CTAs' windows
    if (relu_in) {
      const int rw = warp - kReluWarp0;
      const int nch = L.win_alloc * (kRB0 + kRB1) / 16;  // chunks per stage (chunk0 rows, then chunk1 rows)
      const int per = (nch / kReluWarps + 31) / 32 * 32;
      const int lo = rw * per < nch ? rw * per : nch, hi = rw == kReluWarps - 1 ? nch : (lo + per < nch ? lo + per : nch);
      const int c1_first = L.win_alloc * kRB0 / 16;   // chunk index where the 64-byte-row block starts
      int j = 0;
      for (int64_t k = local; k < n_ptiles; k += npc, ++j) {
        const int s = j % L.stages;
        mbar_wait(&lfull[s], static_cast<uint32_t>(j / L.stages) & 1u);
        const uint32_t wa = smem_u32(smem + lay.win_off + s * lay.win_stage);
        for (int c0 = lo; c0 < hi; c0 += 32 * 8) {
          uint4 v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = c0 + u * 32 + lane;
            const uint32_t off = c < c1_first ? static_cast<uint32_t>(c) * 16u
                                              : lay.win_c1 + static_cast<uint32_t>(c - c1_first) * 16u;
            if (c < hi) v[u] = lds128(wa + off);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int c = c0 + u * 32 + lane;
            const uint32_t off = c < c1_first ? static_cast<uint32_t>(c) * 16u
                                              : lay.win_c1 + static_cast<uint32_t>(c - c1_first) * 16u;
            v[u].x = relu2<F16>(v[u].x);
            v[u].y = relu2<F16>(v[u].y);
            v[u].z = relu2<F16>(v[u].z);
            v[u].w = relu2<F16>(v[u].w);
            if (c < hi) sts128(wa + off, v[u]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(map_to_rank(&full[s], 0));
      }
    }
  } else if (warp == kStoreWarp) {
    // ------------------------------ TMA store warp (staged launches) ----------
    if (staged && lane == 0) {
      prefetch_tmap(&grp.pout[0]);
      prefetch_tmap(&grp.pout[1]);
      int j = 0;
      for (int64_t k = local; k < n_ptiles; k += npc, ++j) {
        const int64_t tile = 2 * k + rank;
        if (tile >= n_tiles) continue;  // (only ever the last pair tile)
        const int b = tbuf(j);
        mbar_wait(&sfull[b], tpar(j));
        const int32_t row0 = static_cast<int32_t>(tile * 128);
        const uint8_t* rb = smem + lay.rbuf_off + b * kTileBytes;
        tma_store_2d(&grp.pout[0], rb, 0, row0);
        tma_store_2d(&grp.pout[1], rb + 128 * kRB0, 0, row0);
        if (grp.out2) {
          const uint8_t* ob = smem + lay.o2_off;
          tma_store_2d(&grp.pout2[0], ob, 0, row0);
          tma_store_2d(&grp.pout2[1], ob + 128 * kRB0, 0, row0);
        }
        bulk_commit();
        bulk_wait_read0();  // the buffers may be rewritten once the stores have read them
        mbar_arrive(&rempty[b]);
        if (grp.out2) mbar_arrive(o2free);
      }
      bulk_wait0();
    }
  } else {
    // ------------------------------ epilogue (warps 2..9, both CTAs) ----------
    // Two warps per TMEM lane quadrant (48 channels each); the warp's 48 accumulator columns are read at
    // once and the accumulator released before any arithmetic.  Unstaged (conv1: one output, no
    // residual): 32-byte global stores per row.  Staged (residual and/or second output): the residual
    // comes from the TMA-loaded tile buffer, y is written back in place and the pre-activated copy into
    // o2buf (16-byte swizzled shared stores), and the store warp issues the TMA stores.
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int q = warp & 3;
    const int hh = (warp - 2) >> 2;  // channel half [48 hh, 48 hh + 48)
    const PlaneGeom geo = L.geo;
    const uint32_t tempty_leader0 = map_to_rank(&tempty[0], 0);
    const uint32_t tempty_leader1 = map_to_rank(&tempty[1], 0);
    const uint32_t rbuf_a = smem_u32(smem + lay.rbuf_off);
    const uint32_t o2_a = smem_u32(smem + lay.o2_off);
    const uint32_t trow = static_cast<uint32_t>(q * 32 + lane);  // this thread's row in the tile
    int j = 0;
    for (int64_t k = local; k < n_ptiles; k += npc, ++j) {
      const int a = j & 1, b = tbuf(j);
      const int64_t tile = 2 * k + rank;
      const bool live = tile < n_tiles;
      const int64_t p = tile * 128 + trow;
      u32x8 rres[3];  // unstaged: this row's residual, fetched before the accumulator wait
      if (!staged && grp.res && live) {
        const __nv_bfloat16* rrow = grp.res + p * kC + 48 * hh;
#pragma unroll
        for (int i = 0; i < 3; ++i) rres[i] = ldg256(rrow + 16 * i);
      }
      mbar_wait(&tfull[a], static_cast<uint32_t>(j >> 1) & 1u);
      tc_fence_after();
      const bool valid = live && geo.valid(p);
      const uint32_t taddr = tbase + static_cast<uint32_t>(a * kC + 48 * hh) + (static_cast<uint32_t>(q * 32) << 16);
      uint32_t r[48];
      tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
      tmem_ld16(taddr + 32, *reinterpret_cast<uint32_t(*)[16]>(r + 32));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive_relaxed(&tempty[a]);
        else
          mbar_arrive_cluster_relaxed(a ? tempty_leader1 : tempty_leader0);
      }
      if (!live) continue;  // (only ever the last pair tile)
      if (staged) {
        if (grp.res)
          mbar_wait(&rfull[b], tpar(j));
        else
          mbar_wait(&rempty[b], tpar(j) ^ 1u);
        if (grp.out2) mbar_wait(o2free, (static_cast<uint32_t>(j) & 1u) ^ 1u);
      }
      const uint32_t rb = rbuf_a + static_cast<uint32_t>(b) * kTileBytes;
      __nv_bfloat16* orow = grp.out ? grp.out + p * kC : nullptr;
      __nv_bfloat16* orow2 = grp.out2 ? grp.out2 + p * kC : nullptr;
#pragma unroll
      for (int pc = 0; pc < 3; ++pc) {
        const int c0 = 48 * hh + 16 * pc;
        const uint32_t off0 = tile_off(trow, static_cast<uint32_t>(c0));
        const uint32_t off1 = tile_off(trow, static_cast<uint32_t>(c0 + 8));
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[16 * pc + i]) + s_bias[c0 + i];
        if (grp.res) {  // staged: the residual rows arrived by TMA in the tile buffer
          uint4 rv[2];
          if (staged) {
            rv[0] = lds128(rb + off0);
            rv[1] = lds128(rb + off1);
          } else {
            rv[0] = make_uint4(rres[pc].v[0], rres[pc].v[1], rres[pc].v[2], rres[pc].v[3]);
            rv[1] = make_uint4(rres[pc].v[4], rres[pc].v[5], rres[pc].v[6], rres[pc].v[7]);
          }
          const uint32_t* rp = reinterpret_cast<const uint32_t*>(rv);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 f = unpack2<F16>(rp[i]);
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
        u32x8 o;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o.v[i] = pack2<F16>(v[2 * i], v[2 * i + 1]);
        }
        if (staged) {
          sts128(rb + off0, make_uint4(o.v[0], o.v[1], o.v[2], o.v[3]));
          sts128(rb + off1, make_uint4(o.v[4], o.v[5], o.v[6], o.v[7]));
        } else if (orow) {
          stg256(orow + c0, o);
        }
        if (orow2) {
          u32x8 o2;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float x0 = fmaxf(v[2 * i] * s_s2[c0 + 2 * i] + s_t2[c0 + 2 * i], 0.f);
            const float x1 = fmaxf(v[2 * i + 1] * s_s2[c0 + 2 * i + 1] + s_t2[c0 + 2 * i + 1], 0.f);
            o2.v[i] = pack2<F16>(valid ? x0 : 0.f, valid ? x1 : 0.f);
          }
          if (staged) {
            sts128(o2_a + off0, make_uint4(o2.v[0], o2.v[1], o2.v[2], o2.v[3]));
            sts128(o2_a + off1, make_uint4(o2.v[4], o2.v[5], o2.v[6], o2.v[7]));
          } else {
            stg256(orow2 + c0, o2);
          }
        }
      }
      if (staged) {
        fence_proxy_async_smem();  // generic stores -> the TMA store's async-proxy reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfull[b]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its peer may still signal its barriers
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(kTmemCols) : "memory");
}

}  // namespace

bool conv_pair96_supported(int cin, int cout, int ks, int halo) {
  return cin == kC && cout == kC && ks == 3 && conv_pair96_stages(((128 + 2 * halo) + 31) / 32 * 32, false) > 0;
}

int conv_pair96_stages(int win_alloc, bool staged) {
  for (int st = staged ? 2 : 4; st >= 2; --st)
    if (pair_layout(st, win_alloc, staged).total <= 227u * 1024u) return st;
  return 0;
}

size_t conv_pair96_smem_bytes(int stages, int win_alloc, bool staged) { return pair_layout(stages, win_alloc, staged).total; }

const char* conv_pair96_launch(const TcLaunch& L, int num_sms, cudaStream_t stream) {
  const PairLayout lay = pair_layout(L.stages, L.win_alloc, (L.flags & kPairStaged) != 0);
  auto kern = L.fp16 ? conv_pair96_kernel<true> : conv_pair96_kernel<false>;
  ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(lay.total));
  const int64_t pair_work = static_cast<int64_t>(L.ngroups) * ((L.geo.n_tiles + 1) / 2);
  int pairs = static_cast<int>(pair_work < num_sms / 2 ? pair_work : num_sms / 2);
  if (pairs < L.ngroups) pairs = L.ngroups;
  launch_pdl(kern, dim3(2 * pairs), dim3(kThreads), lay.total, stream, L);
  if (L.flags & kPairReluIn) return L.fp16 ? "conv_pair96_kernel<f16,relu_in>" : "conv_pair96_kernel<relu_in>";
  return L.fp16 ? "conv_pair96_kernel<f16>" : "conv_pair96_kernel";
}

}  // namespace cnrx
