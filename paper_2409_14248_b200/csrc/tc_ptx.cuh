// tc_ptx.cuh -- thin inline-PTX wrappers for the sm_100a tensor-core path: mbarriers, the 1-D
// bulk async copy (UBLKCP) and L2 prefetch, 3-D TMA loads, TMEM allocation, tcgen05.mma (kind::f16
// with BF16 operands and F32 accumulate, cta_group::1), tcgen05.commit / ld / st, bf16 hi/lo splits
// and packed fp32 pair arithmetic (FFMA2 / FMUL2).  Descriptor bit layouts follow the sm_100 UMMA formats
// (shared-memory matrix descriptor and 32-bit instruction descriptor).
#pragma once
#include <cstdint>
#include <cuda.h>            // CUtensorMap (type only; the encoder is fetched through the runtime)
#include <cuda_runtime.h>

namespace hrkan {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait suspends the waiting warp until the phase completes or this many ns pass (instead of the
// short default window), so waiting warps stop stealing issue slots from the generator warps.
#ifndef MBAR_SUSPEND_NS
#define MBAR_SUSPEND_NS 0
#endif
// Hang guard (debug builds, -DHRKAN_HANG_GUARD=1): every wait is bounded by
// HRKAN_HANG_CYCLES SM clock cycles (default 2^34, ~9 s at 1.9 GHz).  A wait that runs out prints the
// block, thread, barrier and parity and executes a trap, so a barrier-phase bug surfaces as a launch
// failure (HRKAN_ECUDA on the next call) instead of a hung GPU.  Production builds keep the unbounded
// spin (no clock reads in the hot loops).
#ifndef HRKAN_HANG_GUARD
#define HRKAN_HANG_GUARD 0
#endif
#ifndef HRKAN_HANG_CYCLES
#define HRKAN_HANG_CYCLES (1ll << 34)
#endif
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
static __device__ __noinline__ void hang_trap(uint64_t* bar, uint32_t parity) {
  printf("hrkan hang guard: block (%d,%d,%d) thread %d waited > %lld cycles on mbarrier smem+0x%x parity %u\n",
         (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x, (long long)HRKAN_HANG_CYCLES,
         smem_u32(bar), parity);
  __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if HRKAN_HANG_GUARD
  const long long t0 = clock64();
  while (!mbar_try(bar, parity))
    if (clock64() - t0 > (long long)HRKAN_HANG_CYCLES) hang_trap(bar, parity);
#elif MBAR_SUSPEND_NS == 0
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(MBAR_SUSPEND_NS)
      : "memory");
#endif
}

// Producer-side arrival of a warp's generic-proxy smem writes: every lane fences its writes to the
// async proxy, the warp converges, one lane arrives (HRKAN_WARP_ARRIVE) -- the barrier then counts
// warps, not threads (32x fewer arrive operations on the stage barrier).  Without the switch every
// thread arrives.
#ifndef HRKAN_WARP_ARRIVE
#define HRKAN_WARP_ARRIVE 0
#endif
constexpr unsigned ARRIVALS_PER_WARP = HRKAN_WARP_ARRIVE ? 1u : 32u;
__device__ __forceinline__ void fence_proxy_async_smem();
__device__ __forceinline__ void warp_arrive_after_writes(uint64_t* bar) {
  fence_proxy_async_smem();
#if HRKAN_WARP_ARRIVE
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
#else
  mbar_arrive(bar);
#endif
}

// ------------------------------------------------------------------ packed fp32 pairs (sm_100 FFMA2/FMUL2)
// Two lanes of fp32 arithmetic per instruction; the pair lives in a 64-bit register pair.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float max_nan(float a, float b) {   // NaN-propagating max
  float d;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
  return d;
}

// generic-proxy smem writes -> visible to the async proxy (tensor core / bulk copy)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------------ bulk copy global -> smem
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// L2 prefetch of a contiguous global range (16-B aligned, multiple of 16 bytes); no completion.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}

// ------------------------------------------------------------------ TMA tensor copy global -> smem
// 3-D tiled box (coordinates innermost first); out-of-bounds elements are zero-filled and still
// count towards the transaction bytes.
__device__ __forceinline__ void tma_load_3d(void* dst_smem, const CUtensorMap* tmap, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a 3-D tensor box (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* tmap, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// ------------------------------------------------------------------ TMEM
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {   // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {      // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ------------------------------------------------------------------ descriptors
// Shared-memory matrix descriptor, SWIZZLE_NONE (interleaved core matrices of 8 rows x 16 B):
//   bits [0,14) start>>4, [16,30) LBO>>4, [32,46) SBO>>4, [46,48) version=1, [61,64) layout=0.
// K-major: LBO = byte distance between the two 16-B K-chunks of one MMA, SBO = between 8-row
// groups.  MN-major: LBO = between 8-deep K groups... (see each kernel for the layout it uses).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // version (sm_100)
  return d;                 // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE
}


// D[tmem] (+)= A[smem] * B[smem]^T   (single elected thread)

// Instruction descriptor kind::f16 with BF16 A/B (K-major) and an F32 accumulator.
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4)            // c_format F32
         | (1u << 7)          // a_format BF16
         | (1u << 10)         // b_format BF16
         | ((N >> 3) << 17) | ((M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, BF16 operands, K = 16 per instruction (single elected thread)
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// mbarrier arrives when all previously issued tcgen05.mma of this thread have completed
// Warp-wide forms: the WHOLE warp executes the issue loop (convergent control flow, so the compiler keeps
// the loop's descriptors and addresses in uniform registers) and one lane elected inside the asm issues the
// tcgen05 instruction.  Issued from a lane-0-only branch instead, every UTCHMMA is wrapped in a uniformising
// loop of ELECT + 5 R2UR (measured ~80 cycles per MMA: the issue, not the tensor core, bounded N = 64 tiles).
__device__ __forceinline__ void mma_bf16_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 bit, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 16 consecutive columns per thread (store); complete with tmem_st_wait()
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// named barrier among `nthreads` threads (id 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// bf16x3 split: x = hi + lo + r with hi = bf16_rn(x), lo = bf16_rn(x - hi),
// |r| <= 2^-18 |x|; a*b ~ ah*bh + ah*bl + al*bh (the dropped al*bl is <= 2^-18 |ab|).
// Pairs are packed little-endian: the element at the lower K index sits in the low 16 bits.
__device__ __forceinline__ uint32_t pack_bf16x2(float e0, float e1) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(e1), "f"(e0));
  return r;
}
__device__ __forceinline__ void split2_bf16(float e0, float e1, uint32_t& hi, uint32_t& lo) {
  hi = pack_bf16x2(e0, e1);
  const float r0 = e0 - __uint_as_float(hi << 16);
  const float r1 = e1 - __uint_as_float(hi & 0xFFFF0000u);
  lo = pack_bf16x2(r0, r1);
}
__device__ __forceinline__ void split4_bf16(float4 v, uint2& hi, uint2& lo) {
  split2_bf16(v.x, v.y, hi.x, lo.x);
  split2_bf16(v.z, v.w, hi.y, lo.y);
}
__device__ __forceinline__ void split8_bf16(const float (&v)[8], uint4& hi, uint4& lo) {
  split2_bf16(v[0], v[1], hi.x, lo.x);
  split2_bf16(v[2], v[3], hi.y, lo.y);
  split2_bf16(v[4], v[5], hi.z, lo.z);
  split2_bf16(v[6], v[7], hi.w, lo.w);
}
// host/device scalar version for weight tiling: returns the two bf16 bit patterns
__device__ __forceinline__ void split1_bf16(float x, uint16_t& hi, uint16_t& lo) {
  const uint32_t h = pack_bf16x2(x, 0.f);
  hi = (uint16_t)(h & 0xFFFFu);
  const uint32_t l = pack_bf16x2(x - __uint_as_float(h << 16), 0.f);
  lo = (uint16_t)(l & 0xFFFFu);
}

}  // namespace tc
}  // namespace hrkan
