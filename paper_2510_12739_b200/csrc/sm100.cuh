// sm100.cuh — thin inline-PTX layer for the sm_100a features the CoNet-Rx kernels use:
// mbarriers, TMA (tensor + bulk copies), tcgen05 (TMEM alloc / UMMA / commit / ld) and the
// shared-memory matrix descriptors. Everything here is device-side and header-only.
//
// Conventions:
//   * A and B operands are K-major with the 128-byte swizzle (one 128 B row = 64 bf16 channels),
//     stored as rows of 128 B, 8-row atoms of 1024 B (SBO = 1024 B).
//   * 32-channel tails use the 64-byte swizzle (rows of 64 B, 8-row atoms of 512 B).
//   * The conv kernels address the A operand at ARBITRARY row offsets inside a TMA-loaded window
//     (the 3x3 taps are row shifts of the flattened activation plane). The descriptor's base-offset
//     field carries the row phase inside the swizzle atom; tools/probes/umma_probe.cu pins the
//     semantics on hardware.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

namespace cnrx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------------------------------------
// mbarrier
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Arrive without release semantics: for "accumulator drained" signals, whose only precondition (the
// TMEM loads completed, tcgen05.wait::ld + fence::before_thread_sync) does not involve memory; a
// release arrive would first wait for the warp's outstanding shared / global stores.
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
#ifndef CNRX_WAIT_HINT_NS
#define CNRX_WAIT_HINT_NS 0
#endif
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
#if CNRX_WAIT_HINT_NS > 0
  // suspend-time hint: a waiting warp sleeps (no issue slots, no power) until the phase completes
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "n"(CNRX_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}

// Bounded wait: a protocol bug must surface as a trapped kernel (a CUDA error on the host), never as a
// GPU that spins forever. ~8e9 cycles is several seconds at any clock the B200 runs at.
#ifndef CNRX_WAIT_LIMIT_CYCLES
#define CNRX_WAIT_LIMIT_CYCLES 8000000000ull
#endif
// A timed-out wait traps (the host sees cudaErrorLaunchFailure).  The diagnostic printf is a debug build
// option (-DCNRX_WAIT_PRINTF): inlined at every wait site it gave the production kernels a 48-byte stack
// frame and local-memory traffic.
__device__ __forceinline__ void wait_timeout(uint32_t parity) {
#ifdef CNRX_WAIT_PRINTF
  printf("cnrx: mbarrier wait timeout (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x, parity);
#else
  (void)parity;
#endif
  __trap();
}
// The clock is checked once per 16 polls: a spinning warp's issue slots are shared with the warps doing
// the work (polls were ~25 % of the fused block kernel's issued instructions with a check per poll).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  for (;;) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (mbar_try_wait(addr, parity)) return;
    if (static_cast<unsigned long long>(clock64() - t0) > CNRX_WAIT_LIMIT_CYCLES) wait_timeout(parity);
  }
}

// Bounded wait with cluster-scope acquire: for barriers other CTAs of the cluster arrive on with
// release.cluster semantics (their shared-memory writes must be visible to this CTA's UMMAs).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  auto try_once = [&]() {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
  };
  if (try_once()) return;
  const long long t0 = clock64();
  for (;;) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (try_once()) return;
    if (static_cast<unsigned long long>(clock64() - t0) > CNRX_WAIT_LIMIT_CYCLES) wait_timeout(parity);
  }
}

// Same, but polling with a nanosleep back-off: for kernels with many waiting warps, whose polls would
// otherwise take issue slots from the working ones (a try_wait returns after a few tens of cycles).
template <unsigned kSleepNs>
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  for (;;) {
    __nanosleep(kSleepNs);
    if (mbar_try_wait(addr, parity)) return;
    if (static_cast<unsigned long long>(clock64() - t0) > CNRX_WAIT_LIMIT_CYCLES) wait_timeout(parity);
  }
}

// ---------------------------------------------------------------------------------------------
// Async proxy fences and TMA
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// 2-D tiled TMA load; coordinates are (inner, outer) in elements, may be negative / out of bounds
// (the hardware zero-fills).
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Plain (non-tensor) bulk copy global -> shared, completes on an mbarrier. 16 B aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(gsrc)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Plain bulk copy shared -> global (bulk_group completion, like tma_store_2d).  16 B aligned, size % 16 == 0.
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(gdst)),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}

// ---------------------------------------------------------------------------------------------
// tcgen05 / TMEM
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 or fp16 in, per the idesc; fp32 accumulate). Issued by one thread.
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16: A (M x 16 bf16) lives in TMEM (lane = row, 8 columns
// of packed bf16 pairs per K=16 step).
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Same, the B descriptor given as its two 32-bit halves (joined inside the asm): issuers that walk a
// window at many row offsets keep one 32-bit offset per tap instead of a hoisted 64-bit descriptor per
// (tap, K step) -- the hoisted form spilled in the fused block kernel's issuer (80-register cap).
__device__ __forceinline__ void umma_f16_ts_lohi(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n .reg .b64 bd;\n setp.ne.b32 p, %5, 0;\n mov.b64 bd, {%2, %3};\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], bd, %4, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}

// SS form with both descriptors given as 32-bit halves: the low word of a K-major smem descriptor is
// (address >> 4) | (1 << 16), so an issuer walking a window keeps one 32-bit base per operand and adds
// (row * row_bytes + k_bytes) / 16 per UMMA -- one IADD instead of rebuilding a 64-bit descriptor.
__device__ __forceinline__ uint32_t sdesc_hi(uint32_t sbo, uint32_t swizzle) {
  return ((sbo >> 4) & 0x3FFFu) | (1u << 14) | ((swizzle & 7u) << 29);
}
__device__ __forceinline__ uint32_t sdesc_lo(uint32_t addr) { return ((addr >> 4) & 0x3FFFu) | (1u << 16); }
__device__ __forceinline__ void umma_ss_lohi(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n .reg .b64 ad, bd;\n setp.ne.b32 p, %6, 0;\n mov.b64 ad, {%1, %2};\n mov.b64 bd, {%3, %4};\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], ad, bd, %5, p;\n}\n" ::"r"(d_tmem),
      "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}

// registers -> TMEM: 32 lanes x 32 bit, 8 consecutive columns (lane quadrant fixed by warp % 4).
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Arrive (once) on an mbarrier when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Instruction descriptor: bf16 x bf16 -> fp32, both operands K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N) {
  return (1u << 4)            // D format = f32
         | (1u << 7)          // A format = bf16
         | (1u << 10)         // B format = bf16
         | ((N >> 3) << 17)   // N / 8
         | ((M >> 4) << 24);  // M / 16
}

enum : uint32_t { kSwizzleNone = 0, kSwizzle128 = 2, kSwizzle64 = 4, kSwizzle32 = 6 };

// Shared-memory matrix descriptor (tcgen05 / sm_100 format, version 1).
//   start: smem byte address of the first row (16 B aligned)
//   sbo:   byte distance between consecutive 8-row groups (1024 for SW128 rows of 128 B)
//   base_offset: row phase (0..7) of `start` inside the swizzle pattern.
__device__ __forceinline__ uint64_t make_sdesc(uint32_t start, uint32_t sbo, uint32_t swizzle,
                                               uint32_t base_offset) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((start >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;  // LBO (unused for swizzled K-major; canonical value 1)
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;  // descriptor version for sm_100
  d |= static_cast<uint64_t>(base_offset & 7u) << 49;
  d |= static_cast<uint64_t>(swizzle & 7u) << 61;
  return d;
}

// TMEM -> registers: 32 lanes x 32 bit, 32 consecutive columns. Lane quadrant is fixed by warp % 4.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Byte offset of (row, 16-byte chunk) inside a 128B-swizzled K-major tile whose base is 1024 B aligned.
__host__ __device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t chunk) {
  return row * 128u + ((chunk ^ (row & 7u)) << 4);
}
// Same for the 64B swizzle (rows of 64 B, 4 chunks, pattern repeats every 8 rows / 512 B).
__host__ __device__ __forceinline__ uint32_t sw64_offset(uint32_t row, uint32_t chunk) {
  return row * 64u + ((chunk ^ ((row >> 1) & 3u)) << 4);
}


// %globaltimer in ns (debug tracing: effective SM clock = clock64 cycles / elapsed ns)
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace slots 12..15: CTA count, ~min start, max end, summed CTA ns (see api.cpp trace printing)
__device__ __forceinline__ void trace_cta_window(unsigned long long* tr, unsigned long long g_start) {
  const unsigned long long g_end = globaltimer_ns();
  atomicAdd(&tr[12], 1ull);
  atomicMax(&tr[13], ~g_start);
  atomicMax(&tr[14], g_end);
  atomicAdd(&tr[15], g_end - g_start);
}

// TMEM -> registers, 16 lanes x 256 bit, 4 repetitions along columns (CuTe SM100_TMEM_LOAD_16dp256b4x):
// thread t gets r[4i + 0/1] = (lane t/4, columns 8i + 2(t%4) + 0/1), r[4i + 2/3] = lane t/4 + 8, same columns.
__device__ __forceinline__ void tmem_ld16x256b_x4(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
// Four 8x8 b16 matrices, transposed: thread a supplies the address of row a%8 of matrix a/8 (16 bytes);
// thread t gets r[i] = (rows 2(t%4), 2(t%4)+1 ; column t/4) of matrix i, low half = the even row.
__device__ __forceinline__ void ldsm_x4_trans(uint32_t saddr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(saddr)
               : "memory");
}
// Inverse of ldsm_x4_trans: r[i] holds (rows 2(t%4), 2(t%4)+1 ; column t/4) of matrix i.
__device__ __forceinline__ void stsm_x4_trans(uint32_t saddr, const uint32_t (&r)[4]) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.trans.shared.b16 [%0], {%1,%2,%3,%4};"
               :
               : "r"(saddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}

// TMEM -> registers: 32 lanes x 32 bit, 8 consecutive columns.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
}

// ---------------------------------------------------------------------------------------------
// 1x1 LLR head on the tensor core (head.cu for 64-channel planes, conv_ws.cu's fused-head epilogue):
// the folded interaction z of a 128-row tile, rounded to bf16 and stored K-major with the 128-byte
// swizzle ([128 rows][64 ch], exactly the layout of a staged output tile), times the head weights
// [16 outputs (nb real, rest zero)][64 ch] bf16 (same layout) -> D [128 lanes = rows][16 fp32 columns].
// Both kernels issue the same four K=16 UMMAs per row, so a row's LLRs do not depend on which
// kernel (or which TMEM lane) computed them.
// ---------------------------------------------------------------------------------------------
constexpr int kHeadTcN = 16;
constexpr uint32_t kHeadTcWBytes = kHeadTcN * 128;
__device__ __forceinline__ void head_tc_pack_weights(uint8_t* hw, const float* w, int nb, int tid, int nthreads) {
  for (int e = tid; e < kHeadTcN * 64; e += nthreads) {
    const int n = e >> 6, c = e & 63;
    const float v = n < nb ? w[c * nb + n] : 0.f;
    *reinterpret_cast<__nv_bfloat16*>(hw + n * 128 + ((((c >> 3) ^ (n & 7))) << 4) + (c & 7) * 2) =
        __float2bfloat16(v);
  }
}
__device__ __forceinline__ void head_tc_umma(uint32_t d_tmem, uint32_t z_addr, uint32_t hw_addr) {
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((kHeadTcN >> 3) << 17) | ((128u >> 4) << 24);
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
    umma_f16(d_tmem, make_sdesc(z_addr + kk * 32, 1024, kSwizzle128, 0), make_sdesc(hw_addr + kk * 32, 1024, kSwizzle128, 0),
              idesc, kk > 0 ? 1u : 0u);
}

// ---------------------------------------------------------------------------------------------
// clusters
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared-memory object in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cl_map(const void* p, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(smem_u32(p)), "r"(rank));
  return d;
}
// Remote arrivals are relaxed: a release.cluster arrive first waits until every global store the warp
// issued before it is visible cluster-wide (e.g. the fused head's LLR stores), while the only thing
// these signals order is shared-memory reuse whose reads / async copies have already completed.
__device__ __forceinline__ void cl_arrive(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void cl_arrive_expect_tx(uint32_t cluster_bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_bar), "r"(bytes)
               : "memory");
}
// wait for a phase of a local barrier that remote CTAs arrive on (acquire at cluster scope)
__device__ __forceinline__ void cl_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
}
// bulk copy of this CTA's shared memory into another CTA's (cluster addresses from cl_map); completion
// (bytes) is signalled on the destination CTA's barrier
__device__ __forceinline__ void bulk_copy_to_cta(uint32_t dst_cluster, const void* src, uint32_t bytes,
                                                 uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(smem_u32(src)), "r"(bytes), "r"(bar_cluster)
               : "memory");
}

// 1024-byte aligned base inside the dynamic shared-memory array.  Offsetting the __shared__ array itself
// (instead of round-tripping through an integer) keeps the pointer in the shared state space, so
// plain loads / stores through it compile to LDS / STS rather than generic LD / ST.
__device__ __forceinline__ uint8_t* smem_align1024(uint8_t* smem_dyn) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dyn));
  return smem_dyn + ((1024u - (a & 1023u)) & 1023u);
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Programmatic dependent launch: let the next kernel in the stream start its prologue (barrier init,
// TMEM allocation, weight staging) on SMs this grid has left, and wait for this grid before touching
// its outputs.  Kernels launched with the PDL attribute must call pdl_wait() before their first
// global read or write of activation data.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// 256-bit global accesses (sm_100: LDG/STG .256): one full 32-byte sector per thread per instruction
struct u32x8 {
  uint32_t v[8];
};
__device__ __forceinline__ u32x8 ldg256(const void* p) {
  u32x8 r;
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]),
                 "=r"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void stg256(void* p, const u32x8& r) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]),
               "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]), "r"(r.v[7])
               : "memory");
}
}  // namespace cnrx
