// head.cu — CoNet-Rx fusion tail + LLR head over 16-bit (bf16 / fp16) activation planes, TMA-streamed.
//
// Replaces the reference's tail of build_conet (network.hpp:520-560): the interaction fusion of the
// main and supplementary subnetwork outputs (elementwise mul / add, network.hpp:526-532, each
// optionally followed by an eval BN, norms.hpp:81-95, and ReLU) and the 1x1 output conv to the LLRs
// (kernels.hpp:47-91 with k = 1), for the left-fold program shape pw_as_fold() recognises.
//
// HBM-bound (it reads every subnet's final plane once: NS x 2C bytes per plane row, writes NB fp32 LLRs
// per RE), so the operand rows are streamed by TMA (128-row boxes; 128-byte swizzle for 64 channels)
// into a shared-memory ring instead of per-thread global loads, which saturated the L1 path at ~3 TB/s.
// Two threads per plane row (C/2 channels each) do the fold and the GEMV in fp32 and combine with one
// shuffle.  C in {64, 96}.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "head.h"
#include "elem16.cuh"
#include "sm100.cuh"

namespace cnrx {

namespace {

constexpr int kHRows = 128;              // rows per tile
constexpr int kConsumers = 256;          // two threads per row, C/2 channels each
constexpr int kThreads = kConsumers + 32;

struct HeadLayout {
  uint32_t ring_off, stage_bytes, aff_off, w_off, b_off, part_off, hw_off, bar_off, total;
};
// tc: the head GEMV runs on the tensor core (64-channel bf16 planes); otherwise on CUDA cores in fp32
__host__ __device__ inline HeadLayout head_layout(int c, int ns, int nb, int stages, bool tc) {
  HeadLayout l{};
  const int kHC = c;
  const uint32_t kPlaneBox = static_cast<uint32_t>(kHRows * c * 2);
  l.ring_off = 0;
  l.stage_bytes = static_cast<uint32_t>(ns) * kPlaneBox;
  uint32_t off = l.stage_bytes * static_cast<uint32_t>(stages);
  l.aff_off = off;
  off += static_cast<uint32_t>(ns) * 2u * kHC * 4u;
  l.w_off = off;
  off += static_cast<uint32_t>(kHC * nb) * 4u;
  l.b_off = off;
  off += 64u;
  l.part_off = off;  // [2][128 rows][nb] partial GEMV sums of the upper channel half (CUDA-core GEMV)
  if (!tc) off += 2u * kHRows * static_cast<uint32_t>(nb) * 4u;
  l.hw_off = off;
  if (tc) {  // tensor-core GEMV: head weight image (1024-aligned); z overwrites the stage's plane 0
    l.hw_off = (off + 1023u) & ~1023u;
    off = l.hw_off + kHeadTcWBytes;
  }
  l.bar_off = (off + 15u) & ~15u;
  l.total = l.bar_off + 2u * 8u * static_cast<uint32_t>(stages) + 16u + 1024u;
  return l;
}

// byte offset of 16-byte chunk `chunk` of row `row` in a TMA tile: 128-byte swizzle for 64-channel rows;
// 96-channel rows are two boxes, channels [0, 64) with the 128-byte swizzle and [64, 96) with the 64-byte
// one (rows wider than a swizzle span; unswizzled 192-byte rows put 16 of a warp's 32 rows on the same
// banks: ncu, cfg3 head at 2 TB/s)
template <int C>
__device__ __forceinline__ uint32_t hoff(uint32_t row, uint32_t chunk) {
  if constexpr (C == 64) return row * 128u + ((chunk ^ (row & 7u)) << 4);
  else if constexpr (C == 96)
    return chunk < 8u ? row * 128u + ((chunk ^ (row & 7u)) << 4)
                      : kHRows * 128u + row * 64u + (((chunk - 8u) ^ ((row >> 1) & 3u)) << 4);
  else return row * static_cast<uint32_t>(C * 2) + (chunk << 4);
}

template <int C, int NB, int NS, bool TC>
__global__ void __launch_bounds__(kThreads, 2) head_tma_kernel(const __grid_constant__ HeadLaunch L) {
  constexpr int kHC = C;
  constexpr int CPT = C / 2;  // channels per thread
  constexpr uint32_t kPlaneBox = kHRows * C * 2;
  extern __shared__ uint8_t smem_dyn[];
  uint8_t* smem = smem_align1024(smem_dyn);
  // 64-channel bf16 planes: the head GEMV runs on the tensor core over the bf16-rounded z tile (the same
  // UMMAs as conv_ws.cu's fused-head epilogue, so both programs give identical LLRs) unless the plan
  // disables it; fp16 plans keep z in fp32 (CUDA-core GEMV): z is a product of subnetwork outputs.
  static_assert(!TC || C == 64, "tensor-core head needs 64-channel planes");
  constexpr bool tc = TC;
  const bool spl = L.split != 0;  // split planes: each operand tile is a (hi, lo) pair of boxes
  const HeadLayout lay = head_layout(C, spl ? 2 * NS : NS, NB, L.stages, tc);
  float* s_aff = reinterpret_cast<float*>(smem + lay.aff_off);  // [NS][2][C]
  float* s_w = reinterpret_cast<float*>(smem + lay.w_off);      // [C][NB]
  float* s_b = reinterpret_cast<float*>(smem + lay.b_off);      // [NB]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + lay.bar_off);
  uint64_t* empty = full + L.stages;
  uint64_t* hdone = empty + L.stages;  // (kTC) head UMMAs of the tile complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hdone + 1);

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < L.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    mbar_init(hdone, 1);
    fence_barrier_init();
  }
  if constexpr (tc) {
    if (tid < 32) tmem_alloc(tmem_slot, 32);
    head_tc_pack_weights(smem + lay.hw_off, L.head_w, NB, tid, kThreads);
    fence_proxy_async_smem();
  }
  for (int e = tid; e < NS * kHC; e += kThreads) {
    const int i = e / kHC, c = e % kHC;
    s_aff[(2 * i) * kHC + c] = L.aff_s[i] ? L.aff_s[i][c] : 1.f;
    s_aff[(2 * i + 1) * kHC + c] = L.aff_t[i] ? L.aff_t[i][c] : 0.f;
  }
  for (int e = tid; e < kHC * NB; e += kThreads) s_w[e] = L.head_w[e];
  if (tid < NB) s_b[tid] = L.head_b[tid];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tc ? *tmem_slot : 0u;
  pdl_trigger();
  pdl_wait();  // PDL: the prologue above overlapped the previous kernel's tail

  const int64_t n_tiles = L.geo.Nalloc / kHRows;
  if (tid >= kConsumers) {
    // ------------------------------ TMA producer ------------------------------
    if (tid == kConsumers) {
      for (int i = 0; i < NS; ++i) prefetch_tmap(&L.maps[i]);
      const uint32_t tx = static_cast<uint32_t>(spl ? 2 * NS : NS) * kPlaneBox;
      int j = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
        const int s = j % L.stages;
        mbar_wait(&empty[s], (static_cast<uint32_t>(j / L.stages) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], tx);
        uint8_t* dst = smem + lay.ring_off + s * lay.stage_bytes;
        const int32_t r0 = static_cast<int32_t>(tile * kHRows);
        for (int i = 0; i < NS; ++i) {
          tma_load_2d(dst + i * kPlaneBox, &L.maps[i], &full[s], 0, r0);
          if (C == 96) tma_load_2d(dst + i * kPlaneBox + kHRows * 128, &L.maps_c1[i], &full[s], 0, r0);
          if (spl) {
            tma_load_2d(dst + (NS + i) * kPlaneBox, &L.lo_maps[i], &full[s], 0, r0);
            if (C == 96) tma_load_2d(dst + (NS + i) * kPlaneBox + kHRows * 128, &L.lo_maps_c1[i], &full[s], 0, r0);
          }
        }
      }
    }
    return;
  }
  // ------------------------------ consumers: two threads per row ------------------
  // warp w covers rows 32*(w/2) .. +31 and channel half w%2, so every shared-memory parameter load
  // (BN tables, head weights) is one broadcast address per warp; the halves meet through smem.
  const int hf = (tid >> 5) & 1, r = (tid & 31) + 32 * (tid >> 6);
  float* s_part = reinterpret_cast<float*>(smem + lay.part_off);
  const PlaneGeom geo = L.geo;
  int j = 0;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++j) {
    const int s = j % L.stages;
    mbar_wait(&full[s], static_cast<uint32_t>(j / L.stages) & 1u);
    const uint8_t* st = smem + lay.ring_off + s * lay.stage_bytes;
    float acc[CPT];
#pragma unroll
    for (int i = 0; i < NS; ++i) {
#pragma unroll
      for (int k = 0; k < CPT / 8; ++k) {
        const uint4 raw = *reinterpret_cast<const uint4*>(st + i * kPlaneBox + hoff<C>(r, (CPT / 8) * hf + k));
        const uint32_t* hv = reinterpret_cast<const uint32_t*>(&raw);
        uint4 rawl = make_uint4(0, 0, 0, 0);
        if (spl) rawl = *reinterpret_cast<const uint4*>(st + (NS + i) * kPlaneBox + hoff<C>(r, (CPT / 8) * hf + k));
        const uint32_t* lv = reinterpret_cast<const uint32_t*>(&rawl);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = unpack2r(L.fp16 != 0, hv[e]);
          if (spl) {  // hi + lo: exact in fp32
            const float2 g = unpack2r(L.fp16 != 0, lv[e]);
            f.x += g.x;
            f.y += g.y;
          }
          const int c = 8 * k + 2 * e;
          if (i == 0) {
            acc[c] = f.x;
            acc[c + 1] = f.y;
          } else if (L.op[i] == PW_MUL) {
            acc[c] *= f.x;
            acc[c + 1] *= f.y;
          } else {
            acc[c] += f.x;
            acc[c + 1] += f.y;
          }
        }
      }
      if (L.aff_s[i]) {
        const float* ps = s_aff + (2 * i) * kHC + CPT * hf;
        const float* pt = s_aff + (2 * i + 1) * kHC + CPT * hf;
#pragma unroll
        for (int c = 0; c < CPT; c += 4) {
          const float4 sv = *reinterpret_cast<const float4*>(ps + c);
          const float4 tv = *reinterpret_cast<const float4*>(pt + c);
          acc[c] = __fmaf_rn(acc[c], sv.x, tv.x);
          acc[c + 1] = __fmaf_rn(acc[c + 1], sv.y, tv.y);
          acc[c + 2] = __fmaf_rn(acc[c + 2], sv.z, tv.z);
          acc[c + 3] = __fmaf_rn(acc[c + 3], sv.w, tv.w);
        }
      }
      if (L.relu[i]) {
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[c] = fmaxf(acc[c], 0.f);
      }
    }
    __syncwarp();
    if constexpr (tc) {
      // z (bf16) overwrites this thread's own chunks of the stage's plane-0 tile (same swizzled layout),
      // one thread issues the head UMMAs, warps 0-3 read TMEM lane quadrants 0-3; the stage is released
      // once the UMMAs have read it
      const uint32_t za = smem_u32(st);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) pk[e] = pack2<false>(acc[8 * k + 2 * e], acc[8 * k + 2 * e + 1]);
        sts128(za + hoff<64>(static_cast<uint32_t>(r), static_cast<uint32_t>(4 * hf + k)), make_uint4(pk[0], pk[1], pk[2], pk[3]));
      }
      fence_proxy_async_smem();
      tc_fence_before();
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
      tc_fence_after();
      if (tid == 0) {
        head_tc_umma(tbase, za, smem_u32(smem + lay.hw_off));
        umma_commit(hdone);
      }
      mbar_wait(hdone, static_cast<uint32_t>(j) & 1u);
      tc_fence_after();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
      const int w = tid >> 5;
      if (w < 4) {
        uint32_t d[8];
        tmem_ld8(tbase + (static_cast<uint32_t>(w * 32) << 16), d);
        tmem_ld_wait();
        const int64_t row = tile * kHRows + w * 32 + (tid & 31);
        if (geo.valid(row)) {
          int b, t, f;
          geo.coords(row, b, t, f);
          float* dst = L.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * NB;
          if constexpr (NB == 4) {
            *reinterpret_cast<float4*>(dst) = make_float4(__uint_as_float(d[0]) + s_b[0], __uint_as_float(d[1]) + s_b[1],
                                                          __uint_as_float(d[2]) + s_b[2], __uint_as_float(d[3]) + s_b[3]);
          } else {
#pragma unroll
            for (int q = 0; q < NB; ++q) dst[q] = __uint_as_float(d[q]) + s_b[q];
          }
        }
      }
      tc_fence_before();
      continue;
    }
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    float part[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) part[q] = 0.f;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const float* wr = s_w + (CPT * hf + c) * NB;
#pragma unroll
      for (int q = 0; q < NB; ++q) part[q] = fmaf(acc[c], wr[q], part[q]);
    }
    float* pb = s_part + ((j & 1) * kHRows + r) * NB;
    if (hf == 1) {
#pragma unroll
      for (int q = 0; q < NB; ++q) pb[q] = part[q];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
    if (hf == 1) continue;
#pragma unroll
    for (int q = 0; q < NB; ++q) part[q] += pb[q];
    const int64_t row = tile * kHRows + r;
    if (geo.valid(row)) {
      int b, t, f;
      geo.coords(row, b, t, f);
      float* dst = L.llr + ((static_cast<int64_t>(b) * geo.T + t) * geo.F + f) * NB;
      if constexpr (NB == 4) {
        *reinterpret_cast<float4*>(dst) =
            make_float4(part[0] + s_b[0], part[1] + s_b[1], part[2] + s_b[2], part[3] + s_b[3]);
      } else if constexpr (NB == 2) {
        *reinterpret_cast<float2*>(dst) = make_float2(part[0] + s_b[0], part[1] + s_b[1]);
      } else {
#pragma unroll
        for (int q = 0; q < NB; ++q) dst[q] = part[q] + s_b[q];
      }
    }
  }
  if constexpr (tc) {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
    tc_fence_after();
    if (tid < 32) tmem_dealloc(tbase, 32);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn_head() {
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

template <int C, int NB, int NS>
void launch_t(const HeadLaunch& L, int stages_bytes_total, cudaStream_t s) {
  // 64-channel heads: tensor-core GEMV (bf16 plans) or CUDA-core fp32 GEMV (fp16 plans / tc_head off)
  constexpr bool kMayTC = C == 64;
  auto kern = (kMayTC && L.tc_head) ? head_tma_kernel<C, NB, NS, kMayTC> : head_tma_kernel<C, NB, NS, false>;
  ensure_smem_attr(reinterpret_cast<const void*>(kern), stages_bytes_total);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_tiles = L.geo.Nalloc / kHRows;
  // two CTAs per SM (16 consumer warps) when they fit, to hide the per-row latency chain
  const int per_sm = stages_bytes_total * 2 + 4096 <= 228 * 1024 ? 2 : 1;
  const int64_t slots = static_cast<int64_t>(per_sm) * sms;
  const unsigned grid = static_cast<unsigned>(n_tiles < slots ? n_tiles : slots);
  launch_pdl(kern, dim3(grid), dim3(kThreads), static_cast<size_t>(stages_bytes_total), s, L);
}

template <int C, int NB>
bool launch_ns(const HeadLaunch& L, int total, cudaStream_t s) {
  switch (L.ns) {
    case 1: launch_t<C, NB, 1>(L, total, s); return true;
    case 2: launch_t<C, NB, 2>(L, total, s); return true;
    case 3: launch_t<C, NB, 3>(L, total, s); return true;
    case 4: launch_t<C, NB, 4>(L, total, s); return true;
    default: return false;
  }
}

template <int C>
bool launch_nb(const HeadLaunch& L, int total, cudaStream_t s) {
  switch (L.nb) {
    case 2: return launch_ns<C, 2>(L, total, s);
    case 4: return launch_ns<C, 4>(L, total, s);
    case 6: return launch_ns<C, 6>(L, total, s);
    case 8: return launch_ns<C, 8>(L, total, s);
    default: return false;
  }
}

}  // namespace

const char* launch_head_tma(const PwProgram& prog, int ns, const int* ops, const int* affs, const int* relus,
                            const PlaneGeom& geo, cudaStream_t s) {
  const int C = prog.C;
  // C in {64, 96} (every BASELINE head); other widths use pointwise.cu's fold kernel
  if ((C != 64 && C != 96) || ns < 1 || ns > kHeadMaxPlanes || geo.Nalloc % kHRows != 0) return nullptr;
  const int nb = prog.head_bits;
  if (nb != 2 && nb != 4 && nb != 6 && nb != 8) return nullptr;
  HeadLaunch L;
  std::memset(&L, 0, sizeof(L));
  L.geo = geo;
  L.ns = ns;
  L.nb = nb;
  L.split = prog.split;
  const int rs = prog.split ? 2 : 1;  // row stride in C-channel units (split rows: [hi C | lo C])
  for (int i = 0; i < ns; ++i) {
    L.op[i] = ops[i];
    L.relu[i] = relus[i];
    L.aff_s[i] = affs[i] >= 0 ? prog.aff_s[affs[i]] : nullptr;
    L.aff_t[i] = affs[i] >= 0 ? prog.aff_t[affs[i]] : nullptr;
    for (int part = 0; part < rs; ++part)
      for (int cb = 0; cb < (C == 96 ? 2 : 1); ++cb) {  // 96 channels: [0, 64) and [64, 96) boxes
        const int bc = C == 96 ? (cb == 0 ? 64 : 32) : C;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(bc), static_cast<cuuint64_t>(geo.Nalloc)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(rs * C * 2)};
        cuuint32_t box[2] = {static_cast<cuuint32_t>(bc), static_cast<cuuint32_t>(kHRows)};
        cuuint32_t es[2] = {1, 1};
        CUtensorMap* m = part == 0 ? (cb == 0 ? &L.maps[i] : &L.maps_c1[i]) : (cb == 0 ? &L.lo_maps[i] : &L.lo_maps_c1[i]);
        const CUtensorMapSwizzle sw = bc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
        CUresult r = encode_fn_head()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                      const_cast<__nv_bfloat16*>(prog.planes[i]) + part * C + cb * 64, dims, strides,
                                      box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw Error(4, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
      }
  }
  L.head_w = prog.head_w;
  L.head_b = prog.head_b;
  L.llr = prog.llr;
  L.fp16 = prog.fp16;
  L.tc_head = prog.tc_head && !prog.fp16 && !prog.split;
  const bool tc = C == 64 && L.tc_head;
  const int nsb = rs * ns;  // operand boxes per tile
  // ring depth: the deepest (<= 3) that still lets two CTAs share an SM (16 consumer warps hide the per-row
  // chains; with one CTA and 96-channel tiles the kernel was latency-bound at 2.5 TB/s), else whatever fits
  // one CTA.  CNRX_HEAD_STAGES (experiments) forces a depth.
  static const int want = std::getenv("CNRX_HEAD_STAGES") ? std::atoi(std::getenv("CNRX_HEAD_STAGES")) : 0;
  int stages = want >= 1 ? want : 3;
  if (want < 1)
    while (stages > 1 && head_layout(C, nsb, nb, stages, tc).total > 113u * 1024u) --stages;
  while (stages > 1 && head_layout(C, nsb, nb, stages, tc).total > 227u * 1024u) --stages;
  L.stages = stages;
  const int total = static_cast<int>(head_layout(C, nsb, nb, stages, tc).total);
  if (total > 227 * 1024) return nullptr;
  bool ok = false;
  switch (C) {
    case 64: ok = launch_nb<64>(L, total, s); break;
    case 96: ok = launch_nb<96>(L, total, s); break;
    default: break;
  }
  return ok ? "head_tma_kernel" : nullptr;
}

}  // namespace cnrx
