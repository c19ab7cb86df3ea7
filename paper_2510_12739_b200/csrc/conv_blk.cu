// conv_blk.cu — one pre-activation residual block in one kernel, conv1's output never leaving the SM:
//
//     h = relu(conv1(relu?(x)) * s2 + t2)        (BN2 folded into conv1's weights and bias)
//     y = conv2(h) + b2 + x
//
// i.e. the MRB block of build_net / append_block (reference network.hpp:451-465: ReLU -> C1 -> BN ->
// ReLU -> C2 -> + skip) over 64-channel 16-bit (bf16 or fp16) planes, 3x3 "same" convolutions (kernels.hpp:47-91).
// The separate-kernel path (conv_ws.cu twice) moves x, h, h, x, y through HBM (4.4 GB per cfg2 block
// at B = 256, conv2 running at ~87 % of the HBM roofline); here only x in and y out (1.8 GB) remain,
// and the block is tensor-core bound.
//
// Both convolutions use conv_ws.cu's weights-stationary form (weights = A operand resident in TMEM,
// two 3x3 taps per UMMA in lane halves, activation window = B operand, partial sums combined in the
// epilogue); see conv_ws.cu and DESIGN.md.  TMEM holds both weight sets (2 x 192 columns), so the
// accumulators are N = 64 columns each (one per convolution, single-buffered): tiles are 63 output rows
// and the tensor core alternates conv1 of one tile with conv2 of an earlier tile, each convolution's
// epilogue draining its accumulator while the other convolution's UMMAs run.
//
// Every CTA owns a contiguous range of tiles, so conv1's output tiles are reused by the conv2 windows
// of neighbouring tiles straight from shared memory: conv1 runs on the range plus one halo tile on each
// side (0.3 % recompute at cfg2 sizes), and its epilogue writes each h row into every conv2 window
// (`W` buffers, 96 rows for T = 14) that contains it.  The residual is read from the x window conv1
// already loaded.
//
// Warp roles (21 warps, 1 CTA per SM):
//   warp 0        TMA producer: x windows (ring of `xstages`)
//   warp 1        conv1 UMMA issuer        warp 19   conv2 UMMA issuer
//   warps 2-9     conv1 epilogue (+ weights -> TMEM at start): TMEM -> combine -> bias, ReLU, zero
//                 padding rows -> bf16/fp16 -> stmatrix into the W windows
//   warps 10-17   conv2 epilogue: TMEM -> combine -> bias + residual (ldmatrix from the x window) ->
//                 bf16/fp16 -> staging -> TMA store of 63 rows
//   warps 18, 20  input ReLU (x window -> relu'd copy, the conv1 B operand) when x is not already
//                 non-negative
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>

#include "conv_blk.h"
#include "kernels.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kC = 64;
constexpr int kRB = 128;          // bytes per plane row
constexpr int kN = 64;            // UMMA N: window rows per instruction
constexpr int kTile = kN - 1;     // output rows per tile (tap B of a pair lands one column later)
constexpr int kPairs = 6;
constexpr int kKSteps = kC / 16;
constexpr int kWCols = kPairs * kKSteps * 8;  // 192 TMEM columns per weight set
constexpr int kAcc1 = 2 * kWCols;              // 384
constexpr int kAcc2 = kAcc1 + kN;              // 448
constexpr int kBox = 32;
#ifndef CNRX_BLK_WSLOTS
#define CNRX_BLK_WSLOTS 5
#endif
constexpr int kWSlots = CNRX_BLK_WSLOTS;  // conv2 windows in flight
// h ring (CNRX_BLK_HRING=1, default): conv1's output rows go into one ring of kWSlots tiles (each row
// stored once) plus a mirror of the ring's first win_rows - 1 rows past its end, so every conv2 window is
// a contiguous row range of the ring; otherwise (0) into kWSlots separate windows (each row stored ~1.5
// times, a third of them through a trash row).  A/B on cfg2 B=256: -3.2 % per block launch
// (profiles/r02_ab_blk_ring.log), bit-identical LLRs.
#ifndef CNRX_BLK_HRING
#define CNRX_BLK_HRING 1
#endif
constexpr int kRingRows = kWSlots * 63;
// warp roles: 0 TMA producer, 1 conv1 UMMA, 2-9 conv1 epilogue, 10-17 conv2 epilogue, 18 and 20 input
// ReLU, 19 conv2 UMMA
// input-ReLU warps: 18 and 20 .. (they copy the window with ReLU applied while the tensor core streams;
// 24 warps keep the same 80-register cap as 21: 6 warps per SM sub-partition either way)
#ifndef CNRX_BLK_RELU_WARPS
#define CNRX_BLK_RELU_WARPS 2
#endif
constexpr int kReluWarps = CNRX_BLK_RELU_WARPS;
constexpr int kWarpE2 = 10, kWarpRelu0 = 18, kWarpMma2 = 19;
constexpr int kThreads = (19 + kReluWarps) * 32;
// fold epilogues (EPI 1 / 2): more warps combine the staged conv2 tile with the fold operand (and run the
// head GEMV), so the conv2-epilogue warps keep their plain per-tile work (7 fold warps: 28 warps, which
// compile to 72 registers without spills)
#ifndef CNRX_BLK_FOLD_WARPS
#define CNRX_BLK_FOLD_WARPS 7
#endif
constexpr int kFoldWarps = CNRX_BLK_FOLD_WARPS, kWarpFold0 = 19 + kReluWarps;
constexpr int kThreadsFold = kThreads + kFoldWarps * 32;
__device__ __forceinline__ int relu_index(int warp) { return warp == kWarpRelu0 ? 0 : warp - 19; }
#ifndef CNRX_BLK_MAXX
#define CNRX_BLK_MAXX 10  // x ring cap; the chooser takes what fits 227 KB (cfg2: 10 stages). 6 -> 10: -1.5 % per launch (profiles/r02m_ab_xring.log)
#endif
constexpr int kMaxXStages = CNRX_BLK_MAXX;

struct BlkLayout {
  uint32_t x_off, stage, xr_off, w_off, stg_off, trash_off, f_off, stg2_off, par_off, bar_off, total;
};
constexpr uint32_t kF32Tile = 64u * 256u;  // one 64-row tile of fp32 channels (fold operand / partial)
// z tile of the fold + head epilogue: rows of 72 floats, channels 32..63 at +36, so the head GEMV's 16-byte
// reads of 16 rows x 2 channel halves per warp spread over all banks
constexpr int kZStride = 72;
constexpr uint32_t kZTile = 64u * kZStride * 4u;
__host__ __device__ constexpr int zidx(int row, int c) { return row * kZStride + (c >= 32 ? c + 4 : c); }
// partial-fold tiles are row-major fp32 [64 rows][64 channels], 16 KB per 63-row output tile
__host__ __device__ inline BlkLayout blk_layout(int xstages, int win_alloc, int relu_in, int epi = 0) {
  BlkLayout s{};
  s.stage = static_cast<uint32_t>(win_alloc * kRB);  // multiple of 4 KB
  s.x_off = 0;
  uint32_t off = s.stage * static_cast<uint32_t>(xstages);
  s.xr_off = off;
  if (relu_in) off += 2u * s.stage;
  s.w_off = off;
  if (CNRX_BLK_HRING)
    off += (static_cast<uint32_t>(kRingRows + win_alloc) * kRB + 1023u) & ~1023u;  // ring + mirror (>= win_rows - 1 rows)
  else
    off += static_cast<uint32_t>(kWSlots) * s.stage;
  s.stg_off = off;                 // 2 x [64 rows][128 B]: the conv2 tile staged for its TMA store / the fold
  off += 2u * 64u * kRB;
  s.trash_off = off;               // 32 rows: destination of stmatrix rows that belong to no window
  off += 32u * kRB;
  s.f_off = off;                   // fold epilogues: 2 operand tiles (16-bit or fp32 rows)
  if (epi) off += 2u * kF32Tile;
  s.stg2_off = off;                // fold epilogues: 2 fp32 partial tiles (EPI 1) / 2 padded z tiles (EPI 2)
  if (epi) off += (2u * (epi == 2 ? kZTile : kF32Tile) + 1023u) & ~1023u;
  s.par_off = off;                 // bias1, bias2; fold: s_prev, t_prev, s, t [64] + head w [64][8], b [8]
  off += 2u * kC * 4u;
  if (epi) off += (4u * kC + kC * 8u + 8u) * 4u;
  s.bar_off = off;                 // 2 * kMaxXStages + 26 mbarriers (46 at 10 stages) + the TMEM address slot: < 512 B
  s.total = off + 512 + 1024;
  return s;
}

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t byte_in_row) {
  return row * 128u + ((((byte_in_row >> 4) ^ (row & 7u)) << 4) | (byte_in_row & 15u));
}

// Copy 16-byte chunks [lo, hi) of a window with ReLU applied (both buffers 1024-byte aligned, same row
// phase, so the 128B swizzle is identical and the copy is chunk for chunk).
template <bool F16>
__device__ __forceinline__ void relu_copy(uint32_t src, uint32_t dst, int lo, int hi, int lane) {
  for (int c0 = lo; c0 < hi; c0 += 32 * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      if (c < hi) v[u] = lds128(src + static_cast<uint32_t>(c) * 16u);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * 32 + lane;
      v[u].x = relu2<F16>(v[u].x);
      v[u].y = relu2<F16>(v[u].y);
      v[u].z = relu2<F16>(v[u].z);
      v[u].w = relu2<F16>(v[u].w);
      if (c < hi) sts128(dst + static_cast<uint32_t>(c) * 16u, v[u]);
    }
  }
}

// Pair-combined accumulator chunk -> four packed 16-bit stmatrix fragments (per 8-channel block `blk`).
// Lanes 16k+i / 16k+8+i of the accumulator hold the tap-A / tap-B partial sums of channel 8k+i; output
// row c = A[c] + B[c+1] (conv_ws.cu).  `xb` is column 32 of this warp's chunk (B of the chunk's last
// row), `res` the residual fragments (or null), `vm` one validity bit per row of the chunk.
template <bool RES, bool RELU, bool F16>
__device__ __forceinline__ void combine_chunk(const uint32_t (&a)[16], uint32_t xb, int blk, float bias,
                                              const uint32_t* res, uint32_t vm, int lane, uint32_t (&o)[4]) {
  const int t0 = lane & 3, ci = lane >> 2;
  const float bnd = __uint_as_float(__shfl_sync(0xffffffffu, xb, 16 * blk + 8 + ci));
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t snd = t0 == 0 ? (i < 3 ? a[4 * (i + 1) + 2] : 0u) : a[4 * i + 2];
    float got = __uint_as_float(__shfl_sync(0xffffffffu, snd, t0 == 3 ? lane - 3 : lane + 1));
    if (i == 3 && t0 == 3) got = bnd;
    float y0 = __uint_as_float(a[4 * i + 0]) + __uint_as_float(a[4 * i + 3]) + bias;
    float y1 = __uint_as_float(a[4 * i + 1]) + got + bias;
    if (RES) {
      const float2 rf = unpack2<F16>(res[i]);
      y0 += rf.x;
      y1 += rf.y;
    }
    if (RELU) {
      y0 = fmaxf(y0, 0.f);
      y1 = fmaxf(y1, 0.f);
    }
    // vm is pre-shifted by 2 * t0 (caller): this thread's rows 8i + 2t0 (+1) are bits 8i (+1)
    if (!((vm >> (8 * i)) & 1u)) y0 = 0.f;
    if (!((vm >> (8 * i + 1)) & 1u)) y1 = 0.f;
    o[i] = pack2<F16>(y0, y1);
  }
}

__device__ __forceinline__ void tmem_ld_x1(uint32_t taddr, uint32_t& r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr) : "memory");
}

__device__ __forceinline__ bool row_valid(const PlaneGeom& geo, int64_t row) { return row >= 0 && geo.valid(row); }

// Accumulator waits of the epilogue warps (16 warps polling): nanosleep back-off of this many ns (0: spin;
// 64 measured -1 % per launch: fewer polls competing for issue slots)
#ifndef CNRX_BLK_EPI_SLEEP_NS
#define CNRX_BLK_EPI_SLEEP_NS 64
#endif
__device__ __forceinline__ void epi_acc_wait(uint64_t* bar, uint32_t parity) {
  if (CNRX_BLK_EPI_SLEEP_NS > 0)
    mbar_wait_backoff<CNRX_BLK_EPI_SLEEP_NS>(bar, parity);
  else
    mbar_wait(bar, parity);
}

template <bool RELU_IN, bool TRACE, bool F16, int EPI>
__global__ void __launch_bounds__(EPI ? kThreadsFold : kThreads, 1) conv_blk64_kernel(const __grid_constant__ BlkLaunch L) {
  constexpr uint32_t IDESC = idesc_e16_f32<F16>(128, kN);
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_align1024(smem_dyn);
  const unsigned long long t_entry = TRACE ? globaltimer_ns() : 0;  // trace: kernel phases (slots 24..27)
  const int XS = L.xstages;
  const BlkLayout lay = blk_layout(XS, L.win_alloc, RELU_IN, EPI);
  float* s_bias1 = reinterpret_cast<float*>(smem + lay.par_off);
  float* s_bias2 = s_bias1 + kC;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* xfull = bars;                   // [XS] x window landed
  uint64_t* xempty = xfull + kMaxXStages;   // [XS] x window consumed (residual read / halo conv1 done)
  uint64_t* xrfull = xempty + kMaxXStages;  // [2] relu'd copy written
  uint64_t* xrempty = xrfull + 2;           // [2] relu'd copy read by conv1
  uint64_t* wfull = xrempty + 2;            // [kWSlots] conv2 window complete
  uint64_t* wempty = wfull + kWSlots;       // [kWSlots] conv2 window read
  uint64_t* t1full = wempty + kWSlots;
  uint64_t* t1empty = t1full + 1;
  uint64_t* t2full = t1empty + 1;
  uint64_t* t2empty = t2full + 1;
  uint64_t* sfull = t2empty + 1;            // [2] staging buffer written by all conv2-epilogue warps
  uint64_t* sfree = sfull + 2;              // [2] staging buffer read by its TMA store
  uint64_t* ffull = sfree + 2;              // [2] fold operand tile landed
  uint64_t* fempty = ffull + 2;             // [2] fold operand tile consumed by all conv2-epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fempty + 2);
  float* s_fold = s_bias2 + kC;             // (EPI) s_prev, t_prev, s, t [64] each, head w [64][8], b [8]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int G = L.ngroups;
  const int g = blockIdx.x % G;
  const int local = blockIdx.x / G;
  const int nct = (static_cast<int>(gridDim.x) - g + G - 1) / G;
  const BlkGroup& grp = L.g[g];
  // contiguous tile range of this CTA; conv1 runs on it plus one tile either side
  const int64_t t_begin = L.n_tiles * local / nct;
  const int64_t t_end = L.n_tiles * (local + 1) / nct;
  const int n_local = static_cast<int>(t_end - t_begin);
  const int U = n_local > 0 ? n_local + 2 : 0;
  const int halo = grp.halo;
  const int win_rows = kN + 2 * halo;  // rows the UMMAs of one window read

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxXStages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);  // conv2's store thread (residual read) or, for halo tiles, conv1's commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&xrfull[s], kReluWarps);  // every ReLU warp
      mbar_init(&xrempty[s], 1);
      mbar_init(&sfull[s], 8);
      mbar_init(&sfree[s], 1);
      mbar_init(&ffull[s], 1);
      mbar_init(&fempty[s], kFoldWarps);
    }
    for (int s = 0; s < kWSlots; ++s) {
      mbar_init(&wfull[s], 8 * 3);  // 8 conv1-epilogue warps x the 3 conv1 tiles a window spans
      mbar_init(&wempty[s], 1);
    }
    mbar_init(t1full, 1);
    mbar_init(t1empty, 8);
    mbar_init(t2full, 1);
    mbar_init(t2empty, 8);
    fence_barrier_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 64 + kC) {
    const int c = threadIdx.x - 64;
    s_bias1[c] = grp.bias1[c];
    s_bias2[c] = grp.bias2[c];
    if (EPI) {
      const BlkFold& fd = L.fold;
      s_fold[c] = fd.s_prev ? fd.s_prev[c] : 1.f;
      s_fold[kC + c] = fd.t_prev ? fd.t_prev[c] : 0.f;
      s_fold[2 * kC + c] = fd.s ? fd.s[c] : 1.f;
      s_fold[3 * kC + c] = fd.t ? fd.t[c] : 0.f;
      if (EPI == 2) {
        for (int q = 0; q < 8; ++q) s_fold[4 * kC + c * 8 + q] = q < fd.nb ? fd.head_w[c * fd.nb + q] : 0.f;
        if (c < 8) s_fold[4 * kC + kC * 8 + c] = c < fd.nb ? fd.head_b[c] : 0.f;
      }
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp >= 2 && warp < 10) {
    // weights -> TMEM: warps 2-5 conv1 (columns [0,192)), warps 6-9 conv2 ([192,384))
    const int q = warp & 3;
    const int set = (warp - 2) >> 2;
    const uint32_t* src = (set == 0 ? grp.wimg1 : grp.wimg2) + static_cast<size_t>(q * 32 + lane) * 8;
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
        tmem_st8(tbase + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(set * kWCols + (b0 + i) * 8), w8[i].v);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (TRACE && threadIdx.x == 0) {
    atomicMax(&L.trace[24], ~t_entry);            // earliest CTA entry
    atomicMax(&L.trace[25], globaltimer_ns());    // latest end of a CTA prologue (barriers, TMEM, weights)
  }
  pdl_trigger();
  pdl_wait();

  const uint32_t x_a = smem_u32(smem + lay.x_off);
  const uint32_t xr_a = smem_u32(smem + lay.xr_off);
  const uint32_t w_a = smem_u32(smem + lay.w_off);
  constexpr bool tr = TRACE;  // per-role cycle counters (CNRX_TRACE): a separate instantiation
  // ring positions advance incrementally (the ring depth XS is a runtime value: no division in the loops)
  auto ring_next = [&](int& slot, uint32_t& phase) {
    if (++slot == XS) {
      slot = 0;
      phase ^= 1u;
    }
  };

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0 && U > 0) {
      prefetch_tmap(&grp.in_map);
      const int nboxes = L.win_alloc / kBox;
      const uint32_t stage_tx = static_cast<uint32_t>(L.win_alloc * kRB);
      long long t_wait = 0;
      int s = 0;
      uint32_t ph = 0;
      for (int u = 0; u < U; ++u, ring_next(s, ph)) {
        const long long t0 = tr ? clock64() : 0;
        mbar_wait(&xempty[s], ph ^ 1u);
        if (tr) t_wait += clock64() - t0;
        mbar_arrive_expect_tx(&xfull[s], stage_tx);
        const int32_t r0 = static_cast<int32_t>((t_begin + u - 1) * kTile - halo);
        uint8_t* win = smem + lay.x_off + s * lay.stage;
        for (int bx = 0; bx < nboxes; ++bx) tma_load_2d(win + bx * kBox * kRB, &grp.in_map, &xfull[s], 0, r0 + bx * kBox);
      }
      if (tr) atomicAdd(&L.trace[kBlkTraceProd], static_cast<unsigned long long>(t_wait));
    }
    if (EPI && lane == 1 && n_local > 0 && !(L.fold.dbg & 1)) {
      // fold operand tiles (one per conv2 tile), double-buffered, consumed by the conv2 epilogue: subnetwork
      // 0's 16-bit rows by TMA, or this tile's 16 KB block of the partial-fold buffer by a plain bulk copy
      const bool f32 = L.fold.opnd_f32 != 0;
      if (!f32) prefetch_tmap(&L.fold.opnd_map);
      for (int v = 0; v < n_local; ++v) {
        const int fb = v & 1;
        mbar_wait(&fempty[fb], (static_cast<uint32_t>(v >> 1) & 1u) ^ 1u);
        uint8_t* dst = smem + lay.f_off + fb * kF32Tile;
        if (f32) {
          mbar_arrive_expect_tx(&ffull[fb], kF32Tile);
          bulk_load(dst, L.fold.opnd_part + static_cast<size_t>(t_begin + v) * (kF32Tile / 4), kF32Tile, &ffull[fb]);
        } else {
          mbar_arrive_expect_tx(&ffull[fb], static_cast<uint32_t>(kTile) * kRB);
          tma_load_2d(dst, &L.fold.opnd_map, &ffull[fb], 0, static_cast<int32_t>((t_begin + v) * kTile));
        }
      }
    }
  } else if (warp == 1 || warp == kWarpMma2) {
    // ------------------------------ UMMA issuers ------------------------------
    // warp 1: conv1 of tiles u = 0 .. U-1; kWarpMma2: conv2 of tiles v = 0 .. n_local-1.  Each warp's
    // tcgen05.commit tracks only its own UMMAs.
    const bool c1 = warp == 1;
    uint32_t shift_b[kPairs];  // byte offset of tap pair p's first window row
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
      const int df = p % 3 - 1;
      const int dt = p < 3 ? -1 : 1;
      shift_b[p] = static_cast<uint32_t>((halo + dt + df * grp.dil * L.geo.T1) * kRB);
    }
    // B descriptor: high half constant (SBO, version, 128B swizzle), low half = start address >> 4 | LBO
    const uint32_t bdesc_hi = static_cast<uint32_t>(make_sdesc(0, 8 * kRB, kSwizzle128, 0) >> 32);
    const uint32_t a_base = tbase + static_cast<uint32_t>(c1 ? 0 : kWCols);
    const uint32_t d_tmem = tbase + static_cast<uint32_t>(c1 ? kAcc1 : kAcc2);
    uint64_t* tfull = c1 ? t1full : t2full;
    uint64_t* tempty = c1 ? t1empty : t2empty;
    const int n = c1 ? U : n_local;
    long long t_in = 0, t_acc = 0;
    const long long t_start = clock64();
    const unsigned long long g_start = globaltimer_ns();
    int s = 0;
    uint32_t ph = 0;
    int ring_pos = kTile - halo;  // (conv2 issuer, h ring) first ring row of window 0
    for (int k = 0; k < n; ++k) {
      uint32_t src;
      uint64_t* release;
      const long long ta = tr ? clock64() : 0;
      if (c1) {
        if (RELU_IN) {
          const int r2 = k & 1;
          mbar_wait(&xrfull[r2], static_cast<uint32_t>(k >> 1) & 1u);
          src = xr_a + static_cast<uint32_t>(r2) * lay.stage;
          release = &xrempty[r2];
        } else {
          mbar_wait(&xfull[s], ph);
          src = x_a + static_cast<uint32_t>(s) * lay.stage;
          release = nullptr;
        }
      } else {
        const int w = k % kWSlots;
        mbar_wait(&wfull[w], static_cast<uint32_t>(k / kWSlots) & 1u);
        if (CNRX_BLK_HRING) {
          // window k = ring rows [((k+1) * 63 - halo) mod R, + win_rows), contiguous through the mirror
          src = w_a + static_cast<uint32_t>(ring_pos) * kRB;
          ring_pos += kTile;
          if (ring_pos >= kRingRows) ring_pos -= kRingRows;
        } else {
          src = w_a + static_cast<uint32_t>(w) * lay.stage;
        }
        release = &wempty[w];
      }
      const long long tb = tr ? clock64() : 0;
      mbar_wait(tempty, (static_cast<uint32_t>(k) & 1u) ^ 1u);
      if (tr) {
        t_in += tb - ta;
        t_acc += clock64() - tb;
      }
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int p = 0; p < kPairs; ++p) {
          const uint32_t row0 = src + shift_b[p];
#pragma unroll
          for (int kk = 0; kk < kKSteps; ++kk)
            umma_f16_ts_lohi(d_tmem, a_base + static_cast<uint32_t>((p * kKSteps + kk) * 8),
                             ((row0 + static_cast<uint32_t>(kk * 32)) >> 4) | (1u << 16), bdesc_hi, IDESC,
                             (p | kk) != 0 ? 1u : 0u);
        }
        if (release) umma_commit(release);
        // halo tiles have no residual reader: their x stage is free once conv1 has read it
        if (c1 && (k == 0 || k == U - 1)) umma_commit(&xempty[s]);
        umma_commit(tfull);
      }
      __syncwarp();
      if (c1) ring_next(s, ph);
    }
    if (tr && lane == 0) {
      atomicAdd(&L.trace[c1 ? kBlkTraceM1In : kBlkTraceM2In], static_cast<unsigned long long>(t_in));
      atomicAdd(&L.trace[c1 ? kBlkTraceM1Acc : kBlkTraceM2Acc], static_cast<unsigned long long>(t_acc));
      if (c1) {
        atomicAdd(&L.trace[kBlkTraceTiles], static_cast<unsigned long long>(n_local));
        atomicAdd(&L.trace[kBlkTraceTotal], static_cast<unsigned long long>(clock64() - t_start));
        trace_cta_window(L.trace, g_start);
      }
    }
  } else if (EPI != 0 && warp >= kWarpFold0) {
    // ------------------------------ interaction fold (EPI 1 / 2) ---------------
    // Per conv2 tile v: the 16-bit y tile the conv2-epilogue warps staged (y rounded exactly as the head
    // kernel would read it from its plane) is combined with the fold operand -- subnetwork 0's 16-bit
    // tile (launch 1, its step-0 BN / ReLU applied) or the previous launch's fp32 partial -- exactly as
    // head.cu folds:  acc = prev (op) y; [fma(acc, s, t)]; [relu].  EPI 1 stores acc (fp32 tile, bulk
    // copy); EPI 2 writes z and runs the 1x1 head, one thread per row, in head.cu's CUDA-core order
    // (fma over channels 0..31 and 32..63 separately, then half 0 + half 1, + bias).
    const int ft = (warp - kWarpFold0) * 32 + lane;  // 0 .. 32 * kFoldWarps - 1
    const BlkFold& fd = L.fold;
    const PlaneGeom geo = L.geo;
    const uint32_t stg_a = smem_u32(smem + lay.stg_off);
    const uint32_t f_a = smem_u32(smem + lay.f_off);
    const float* wf = s_fold + 4 * kC;               // head weights [64][8]
    const float* hb = s_fold + 4 * kC + kC * 8;      // head bias [8]
    int s = XS > 1 ? 1 : 0;  // x stage of conv1 tile u = v + 1 (the residual rows of conv2 tile v)
    uint32_t ph = XS > 1 ? 0u : 1u;
    for (int v = 0; v < n_local; ++v, ring_next(s, ph)) {
      const int sb = v & 1;
      const int64_t p0 = (t_begin + v) * kTile;
      mbar_wait(&sfull[sb], static_cast<uint32_t>(v >> 1) & 1u);
      if (ft == 0) mbar_arrive(&xempty[s]);  // every conv2-epilogue warp read its residual before sfull
      if (!(fd.dbg & 1)) mbar_wait(&ffull[sb], static_cast<uint32_t>(v >> 1) & 1u);
      if (EPI == 1 && ft == 0 && v >= 2) bulk_wait_read1();  // partial tile sb's store (tile v - 2) has read it
      asm volatile("bar.sync 4, %0;" ::"n"(kFoldWarps * 32) : "memory");
      float* out_t = reinterpret_cast<float*>(smem + lay.stg2_off + sb * (EPI == 2 ? kZTile : kF32Tile));
      const uint32_t ys = stg_a + static_cast<uint32_t>(sb) * 64u * kRB;
      const uint32_t fs = f_a + static_cast<uint32_t>(sb) * kF32Tile;
      for (int uu = ft; uu < kTile * 8; uu += kFoldWarps * 32) {
        const int row = uu >> 3, c8 = uu & 7;
        const uint32_t sw = static_cast<uint32_t>(row) * 128u + ((static_cast<uint32_t>(c8) ^ (static_cast<uint32_t>(row) & 7u)) << 4);
        const uint4 yw = lds128(ys + sw);
        const uint32_t yv[4] = {yw.x, yw.y, yw.z, yw.w};
        float prev[8];
        if (fd.opnd_f32) {
          const uint4 a = lds128(fs + static_cast<uint32_t>(row * 256 + c8 * 32));
          const uint4 b = lds128(fs + static_cast<uint32_t>(row * 256 + c8 * 32 + 16));
          prev[0] = __uint_as_float(a.x); prev[1] = __uint_as_float(a.y); prev[2] = __uint_as_float(a.z); prev[3] = __uint_as_float(a.w);
          prev[4] = __uint_as_float(b.x); prev[5] = __uint_as_float(b.y); prev[6] = __uint_as_float(b.z); prev[7] = __uint_as_float(b.w);
        } else {
          const uint4 ow = lds128(fs + sw);  // subnetwork 0's tile, TMA-loaded with the same 128B swizzle
          const uint32_t ov[4] = {ow.x, ow.y, ow.z, ow.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 f = unpack2<F16>(ov[e]);
            prev[2 * e] = f.x;
            prev[2 * e + 1] = f.y;
          }
          if (fd.s_prev) {
#pragma unroll
            for (int e = 0; e < 8; ++e) prev[e] = __fmaf_rn(prev[e], s_fold[8 * c8 + e], s_fold[kC + 8 * c8 + e]);
          }
          if (fd.relu_prev) {
#pragma unroll
            for (int e = 0; e < 8; ++e) prev[e] = fmaxf(prev[e], 0.f);
          }
        }
        float acc[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 y = unpack2<F16>(yv[e]);
          acc[2 * e] = fd.op == PW_MUL ? prev[2 * e] * y.x : prev[2 * e] + y.x;
          acc[2 * e + 1] = fd.op == PW_MUL ? prev[2 * e + 1] * y.y : prev[2 * e + 1] + y.y;
        }
        if (fd.s) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = __fmaf_rn(acc[e], s_fold[2 * kC + 8 * c8 + e], s_fold[3 * kC + 8 * c8 + e]);
        }
        if (fd.relu) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaxf(acc[e], 0.f);
        }
        float* dst = EPI == 2 ? out_t + zidx(row, 8 * c8) : out_t + row * 64 + 8 * c8;
        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
        *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
      if (EPI == 1) fence_proxy_async_smem();  // generic stores -> the bulk store's reads
      __syncwarp();
      if (lane == 0) mbar_arrive(&fempty[sb]);
      asm volatile("bar.sync 4, %0;" ::"n"(kFoldWarps * 32) : "memory");
      if (ft == 0) mbar_arrive(&sfree[sb]);  // the staged y tile is consumed
      if (EPI == 1) {
        if (ft == 0 && !(fd.dbg & 4))
          bulk_store(fd.pout_part + static_cast<size_t>(t_begin + v) * (kF32Tile / 4), out_t, kF32Tile);
        if (ft == 0) bulk_commit();
      } else if (ft < 128) {
        // two threads per row (channel halves), combined with one shuffle: half 0 + half 1, + bias
        const int row = ft >> 1, hf = ft & 1;
        const int64_t prow = p0 + row;
        const int nb = fd.nb;
        float part[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) part[k] = 0.f;
        const float* zr = out_t + zidx(row, 32 * hf);
#pragma unroll 2
        for (int c4 = 0; c4 < 32; c4 += 4) {
          const float4 zq = *reinterpret_cast<const float4*>(zr + c4);
          const float zc[4] = {zq.x, zq.y, zq.z, zq.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4 w0 = *reinterpret_cast<const float4*>(wf + (32 * hf + c4 + u) * 8);
            part[0] = fmaf(zc[u], w0.x, part[0]);
            part[1] = fmaf(zc[u], w0.y, part[1]);
            part[2] = fmaf(zc[u], w0.z, part[2]);
            part[3] = fmaf(zc[u], w0.w, part[3]);
            if (nb > 4) {
              const float4 w1 = *reinterpret_cast<const float4*>(wf + (32 * hf + c4 + u) * 8 + 4);
              part[4] = fmaf(zc[u], w1.x, part[4]);
              part[5] = fmaf(zc[u], w1.y, part[5]);
              part[6] = fmaf(zc[u], w1.z, part[6]);
              part[7] = fmaf(zc[u], w1.w, part[7]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) part[k] += __shfl_xor_sync(0xffffffffu, part[k], 1);
        if (hf == 0 && row < kTile && row_valid(geo, prow) && !(fd.dbg & 2)) {
          int b, t, f;
          geo.coords(prow, b, t, f);
          float* dst = fd.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * nb;
          if (nb == 4) {
            *reinterpret_cast<float4*>(dst) = make_float4(part[0] + hb[0], part[1] + hb[1], part[2] + hb[2], part[3] + hb[3]);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (k < nb) dst[k] = part[k] + hb[k];
          }
        }
      }
    }
    if (EPI == 1 && ft == 0) bulk_wait0();
  } else if (warp == kWarpRelu0 || (warp > kWarpMma2 && warp < 19 + kReluWarps)) {
    // ------------------------------ input ReLU --------------------------------
    if (RELU_IN) {
      const int nchunks = win_rows * (kRB / 16);
      const int per = (nchunks / kReluWarps + 31) / 32 * 32;
      const int ri = relu_index(warp);
      const int lo = ri * per < nchunks ? ri * per : nchunks;
      const int hi = ri == kReluWarps - 1 ? nchunks : (lo + per < nchunks ? lo + per : nchunks);
      long long t_w = 0;
      int s = 0;
      uint32_t ph = 0;
      for (int u = 0; u < U; ++u, ring_next(s, ph)) {
        const int r2 = u & 1;
        const long long t0 = tr ? clock64() : 0;
        mbar_wait(&xfull[s], ph);
        mbar_wait(&xrempty[r2], (static_cast<uint32_t>(u >> 1) & 1u) ^ 1u);
        if (tr) t_w += clock64() - t0;
        relu_copy<F16>(x_a + static_cast<uint32_t>(s) * lay.stage, xr_a + static_cast<uint32_t>(r2) * lay.stage, lo, hi, lane);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xrfull[r2]);
      }
      if (tr && lane == 0 && warp == kWarpRelu0) atomicAdd(&L.trace[kBlkTraceRelu], static_cast<unsigned long long>(t_w));
    }
  } else if (warp < kWarpE2) {
    // ------------------------------ conv1 epilogue (warps 2-9) ----------------
    // warp (q, H): TMEM lane quadrant q (channels 16q .. 16q+15), accumulator columns [32H, 32H+32)
    const int q = warp & 3;
    const int H = ((warp - 2) >> 2) & 1;
    const int ci = lane >> 2;
    const PlaneGeom geo = L.geo;
    float bias[2];
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) bias[blk] = s_bias1[16 * q + 8 * blk + ci];
    const uint32_t trash = smem_u32(smem + lay.trash_off);
    const int r = 32 * H + lane;  // this lane's stmatrix row within the tile
    const uint32_t tq = tbase + kAcc1 + static_cast<uint32_t>(32 * H) + (static_cast<uint32_t>(q * 32) << 16);
    long long t_full = 0, t_w = 0, e1_drain = 0, e1_comb = 0, e1_store = 0, e1_fence = 0;
    int ring_base = 0;  // (h ring) ring row of this tile's first row
    for (int u = 0; u < U; ++u) {
      const int64_t p0 = (t_begin + u - 1) * kTile;
      const uint32_t vm = __ballot_sync(0xffffffffu, row_valid(geo, p0 + r));
      const long long ta = tr ? clock64() : 0;
      epi_acc_wait(t1full, static_cast<uint32_t>(u) & 1u);
      const long long t1 = tr ? clock64() : 0;
      if (tr) t_full += t1 - ta;
      tc_fence_after();
      uint32_t a0[16], a1[16], xb = 0;
      tmem_ld16x256b_x4(tq, a0);
      tmem_ld16x256b_x4(tq + (16u << 16), a1);
      if (H == 0) tmem_ld_x1(tq + 32, xb);  // column 64 would only feed row 63, which no tile owns
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t1empty);
      const long long t2 = tr ? clock64() : 0;
      uint32_t o[2][4];
      combine_chunk<false, true, F16>(a0, xb, 0, bias[0], nullptr, vm >> (2 * (lane & 3)), lane, o[0]);
      combine_chunk<false, true, F16>(a1, xb, 1, bias[1], nullptr, vm >> (2 * (lane & 3)), lane, o[1]);
      if (tr) {
        asm volatile("" ::"r"(o[0][0]), "r"(o[1][3]));  // time the combine, not a sunk copy of it
        const long long t3 = clock64();
        e1_drain += t2 - t1;
        e1_comb += t3 - t2;
      }
      // window u (first written by this tile) must have been released by conv2 of tile u - kWSlots; with
      // the h ring, the rows of tile u - kWSlots this tile overwrites were last read by window u - kWSlots
      const long long tb = tr ? clock64() : 0;
      if (CNRX_BLK_HRING || u < n_local) mbar_wait(&wempty[u % kWSlots], (static_cast<uint32_t>(u / kWSlots) & 1u) ^ 1u);
      const long long tc = tr ? clock64() : 0;
      if (tr) t_w += tc - tb;
      if (CNRX_BLK_HRING) {
        // ring row of h row u * 63 + r (mod R), plus its mirror copy past the ring's end when a window
        // that starts near the end of the ring reads it
        uint32_t pos = static_cast<uint32_t>(ring_base + r);
        if (pos >= static_cast<uint32_t>(kRingRows)) pos -= kRingRows;
        const bool row_ok = r < kTile;
        const bool mir = row_ok && pos < static_cast<uint32_t>(win_rows - 1);
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          const uint32_t cb = static_cast<uint32_t>((2 * q + blk) * 16);
          stsm_x4_trans(row_ok ? w_a + sw128(pos, cb) : trash + sw128(static_cast<uint32_t>(lane), cb), o[blk]);
        }
        if (__any_sync(0xffffffffu, mir)) {
#pragma unroll
          for (int blk = 0; blk < 2; ++blk) {
            const uint32_t cb = static_cast<uint32_t>((2 * q + blk) * 16);
            stsm_x4_trans(mir ? w_a + sw128(pos + kRingRows, cb) : trash + sw128(static_cast<uint32_t>(lane), cb), o[blk]);
          }
        }
        ring_base += kTile;
        if (ring_base >= kRingRows) ring_base -= kRingRows;
      }
      // h row p0 + r belongs to windows v = u-2, u-1, u at window row r + 63 (u-1-v) + halo
#pragma unroll
      for (int dv = -1; dv <= 1 && !CNRX_BLK_HRING; ++dv) {
        const int v = u - 1 + dv;  // dv = -1: v = u - 2 ... dv = +1: v = u
        if (v < 0 || v >= n_local) continue;
        const int wrow = r - dv * kTile + halo;
        const bool mine = r < kTile && wrow >= 0 && wrow < win_rows;
        if (!__any_sync(0xffffffffu, mine)) continue;
        const uint32_t wbase = w_a + static_cast<uint32_t>(v % kWSlots) * lay.stage;
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          const uint32_t cb = static_cast<uint32_t>((2 * q + blk) * 16);
          const uint32_t addr = mine ? wbase + sw128(static_cast<uint32_t>(wrow), cb) : trash + sw128(static_cast<uint32_t>(lane), cb);
          stsm_x4_trans(addr, o[blk]);
        }
      }
      const long long tf = tr ? clock64() : 0;
      fence_proxy_async_smem();
      __syncwarp();
      if (tr) e1_fence += clock64() - tf;
      if (lane == 0) {
#pragma unroll
        for (int dv = -1; dv <= 1; ++dv) {
          const int v = u - 1 + dv;
          if (v >= 0 && v < n_local) mbar_arrive(&wfull[v % kWSlots]);
        }
      }
      if (tr) e1_store += clock64() - tc;
    }
    if (tr && lane == 0 && warp == 2) {
      atomicAdd(&L.trace[kBlkTraceE1Full], static_cast<unsigned long long>(t_full));
      atomicAdd(&L.trace[kBlkTraceE1W], static_cast<unsigned long long>(t_w));
      atomicAdd(&L.trace[kBlkTraceE1Drain], static_cast<unsigned long long>(e1_drain));
      atomicAdd(&L.trace[kBlkTraceE1Comb], static_cast<unsigned long long>(e1_comb));
      atomicAdd(&L.trace[kBlkTraceE1Store], static_cast<unsigned long long>(e1_store));
      atomicAdd(&L.trace[kBlkTraceE1Fence], static_cast<unsigned long long>(e1_fence));
    }
  } else {
    // ------------------------------ conv2 epilogue (warps 10-17) --------------
   {
    // Staging buffers are handed over by mbarriers (no group-wide bar.sync): each warp waits for its
    // buffer to be free, writes its 32 rows x 16 channels, arrives; one thread issues the TMA store.
    const int e = warp - kWarpE2;
    const int q = warp & 3;
    const int H = (e >> 2) & 1;
    const int ci = lane >> 2;
    const PlaneGeom geo = L.geo;
    float bias[2];
#pragma unroll
    for (int blk = 0; blk < 2; ++blk) bias[blk] = s_bias2[16 * q + 8 * blk + ci];
    const bool lead = e == 0 && lane == 0;
    const uint32_t stg_a = smem_u32(smem + lay.stg_off);
    const uint32_t tq = tbase + kAcc2 + static_cast<uint32_t>(32 * H) + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t xrow = static_cast<uint32_t>(halo + 32 * H + lane);
    const uint32_t srow = static_cast<uint32_t>(32 * H + lane);
    const int r = 32 * H + lane;
    if (lead) prefetch_tmap(&grp.out_map);
    long long t_full = 0, e2_drain = 0, e2_comb = 0, e2_store = 0;
    int s = XS > 1 ? 1 : 0;  // x stage of conv1 tile u = v + 1
    uint32_t ph = XS > 1 ? 0u : 1u;
    for (int v = 0; v < n_local; ++v, ring_next(s, ph)) {
      const int64_t p0 = (t_begin + v) * kTile;
      const int sb = v & 1;
      // residual fragments first: the window landed long ago (this wait only orders the TMA writes)
      mbar_wait(&xfull[s], ph);
      const uint32_t xs_a = x_a + static_cast<uint32_t>(s) * lay.stage;
      uint32_t res[2][4];
#pragma unroll
      for (int blk = 0; blk < 2; ++blk) ldsm_x4_trans(xs_a + sw128(xrow, static_cast<uint32_t>((2 * q + blk) * 16)), res[blk]);
      const uint32_t vm = __ballot_sync(0xffffffffu, row_valid(geo, p0 + r));
      const long long ta = tr ? clock64() : 0;
      epi_acc_wait(t2full, static_cast<uint32_t>(v) & 1u);
      const long long t1 = tr ? clock64() : 0;
      if (tr) t_full += t1 - ta;
      tc_fence_after();
      uint32_t a0[16], a1[16], xb = 0;
      tmem_ld16x256b_x4(tq, a0);
      tmem_ld16x256b_x4(tq + (16u << 16), a1);
      if (H == 0) tmem_ld_x1(tq + 32, xb);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t2empty);
      const long long t2 = tr ? clock64() : 0;
      uint32_t o[2][4];
      combine_chunk<true, false, F16>(a0, xb, 0, bias[0], res[0], vm >> (2 * (lane & 3)), lane, o[0]);
      combine_chunk<true, false, F16>(a1, xb, 1, bias[1], res[1], vm >> (2 * (lane & 3)), lane, o[1]);
      long long t3 = 0;
      if (tr) {
        asm volatile("" ::"r"(o[0][0]), "r"(o[1][3]));
        t3 = clock64();
        e2_drain += t2 - t1;
        e2_comb += t3 - t2;
      }
      // staging buffer sb is free once the TMA store of tile v - 2 has read it
      mbar_wait(&sfree[sb], (static_cast<uint32_t>(v >> 1) & 1u) ^ 1u);
      const uint32_t sba = stg_a + static_cast<uint32_t>(sb) * 64u * kRB;
#pragma unroll
      for (int blk = 0; blk < 2; ++blk) stsm_x4_trans(sba + sw128(srow, static_cast<uint32_t>((2 * q + blk) * 16)), o[blk]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[sb]);
      if (EPI == 0 && lead) {  // (fold launches: the fold warps consume the staged tile instead)
        mbar_wait(&sfull[sb], static_cast<uint32_t>(v >> 1) & 1u);
        tma_store_2d(&grp.out_map, smem + lay.stg_off + sb * 64 * kRB, 0, static_cast<int32_t>(p0));
        bulk_commit();
        mbar_arrive(&xempty[s]);  // every warp's residual reads precede its sfull arrival
        if (v >= 1) {
          bulk_wait_read1();      // the store of tile v - 1 has read its staging buffer
          mbar_arrive(&sfree[sb ^ 1]);
        }
      }
      if (tr) e2_store += clock64() - t3;
    }
    if (lead) bulk_wait0();
    if (tr && lead) {
      atomicAdd(&L.trace[kBlkTraceE2Full], static_cast<unsigned long long>(t_full));
      atomicAdd(&L.trace[kBlkTraceE2Drain], static_cast<unsigned long long>(e2_drain));
      atomicAdd(&L.trace[kBlkTraceE2Comb], static_cast<unsigned long long>(e2_comb));
      atomicAdd(&L.trace[kBlkTraceE2Store], static_cast<unsigned long long>(e2_store));
    }
   }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tbase, 512);
  if (TRACE && threadIdx.x == 0) atomicMax(&L.trace[26], globaltimer_ns());  // latest CTA exit
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_blk() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    CNRX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr));
    if (!p) throw Error(4, "cuTensorMapEncodeTiled not available");
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
  CUresult r = encode_fn_blk()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(plane), dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(4, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}


template <bool RELU_IN, bool TRACE, bool F16, int EPI>
void launch_tt(const BlkLaunch& L, int grid, cudaStream_t stream) {
  const BlkLayout lay = blk_layout(L.xstages, L.win_alloc, RELU_IN, EPI);
  ensure_smem_attr(reinterpret_cast<const void*>(conv_blk64_kernel<RELU_IN, TRACE, F16, EPI>), static_cast<int>(lay.total));
  launch_pdl(conv_blk64_kernel<RELU_IN, TRACE, F16, EPI>, dim3(grid), dim3(EPI ? kThreadsFold : kThreads), lay.total,
             stream, L);
}
// the per-role trace counters are a bf16-only debug instantiation; the fold epilogues take a ReLU'd input
// (the last blocks of MRB subnetworks)
template <bool RELU_IN>
void launch_t(const BlkLaunch& L, int grid, cudaStream_t stream) {
  if (RELU_IN && L.epi == 1) {
    if (L.fp16) launch_tt<true, false, true, 1>(L, grid, stream);
    else launch_tt<true, false, false, 1>(L, grid, stream);
  } else if (RELU_IN && L.epi == 2) {
    if (L.fp16) launch_tt<true, false, true, 2>(L, grid, stream);
    else launch_tt<true, false, false, 2>(L, grid, stream);
  } else if (L.epi) {
    throw Error(4, "internal: fused-block fold epilogue needs a ReLU'd block input");
  } else if (L.fp16) {
    launch_tt<RELU_IN, false, true, 0>(L, grid, stream);
  } else if (L.trace) {
    launch_tt<RELU_IN, true, false, 0>(L, grid, stream);
  } else {
    launch_tt<RELU_IN, false, false, 0>(L, grid, stream);
  }
}

}  // namespace

int64_t conv_blk64_tiles(int64_t nalloc) { return (nalloc + kTile - 1) / kTile; }

int conv_blk64_win_alloc(int halo) { return (kN + 2 * halo + kBox - 1) / kBox * kBox; }

// a window may take h rows from at most the neighbouring conv1 tile on either side
bool conv_blk64_supported_halo(int halo) { return halo >= 1 && halo + 1 <= kTile; }

void conv_blk64_make_maps(const void* in, const void* out, int64_t nalloc, BlkGroup* g) {
  make_map(in, nalloc, kBox, &g->in_map);
  make_map(out, nalloc, kTile, &g->out_map);
}

size_t conv_blk64_part_bytes(int64_t nalloc) { return static_cast<size_t>(conv_blk64_tiles(nalloc)) * kF32Tile; }

void conv_blk64_make_fold_maps(const void* opnd, bool opnd_f32, void* pout, int64_t nalloc, BlkFold* f) {
  std::memset(&f->opnd_map, 0, sizeof(f->opnd_map));
  f->opnd_part = nullptr;
  if (opnd_f32)
    f->opnd_part = static_cast<const float*>(opnd);
  else
    make_map(opnd, nalloc, kTile, &f->opnd_map);
  f->pout_part = static_cast<float*>(pout);
  f->opnd_f32 = opnd_f32 ? 1 : 0;
}

size_t conv_blk64_smem_bytes(int xstages, int win_alloc, int relu_in, int epi) {
  return blk_layout(xstages, win_alloc, relu_in, epi).total;
}

int conv_blk64_xstages(int win_alloc, int relu_in, int epi) {
  for (int xs = kMaxXStages; xs >= 4; --xs)
    if (blk_layout(xs, win_alloc, relu_in, epi).total <= 227u * 1024u) return xs;
  return 0;
}

const char* conv_blk64_launch(const BlkLaunch& L, int num_sms, cudaStream_t stream) {
  const int64_t work = static_cast<int64_t>(L.ngroups) * L.n_tiles;
  int grid = static_cast<int>(work < num_sms ? work : num_sms);
  if (grid < L.ngroups) grid = L.ngroups;
  if (L.relu_in)
    launch_t<true>(L, grid, stream);
  else
    launch_t<false>(L, grid, stream);
  return L.epi == 2 ? "conv_blk64_kernel<fold+head>" : L.epi == 1 ? "conv_blk64_kernel<fold>" : "conv_blk64_kernel";
}

}  // namespace cnrx
