// tc.cuh -- minimal sm_100a tcgen05 building blocks (inline PTX): TMEM
// allocation, shared-memory matrix descriptors (K-major, no swizzle), the
// kind::tf32 MMA with fp32 accumulation in TMEM, commit to an mbarrier, and
// TMEM -> register loads.  Layout conventions (PTX ISA "canonical layouts";
// CuTe UMMA::make_umma_desc, K-major INTERLEAVE):
//   an operand tile of R rows (M or N) x K columns (tf32 in 32-bit containers)
//   is stored as 8-row x 16-byte "core matrices": element (r, k) at byte
//     (r / 8) * SBO + (k / 4) * LBO + (r % 8) * 16 + (k % 4) * 4,
//   with LBO = 128 (core matrices adjacent along K) and SBO = (K / 4) * 128.
//   One MMA consumes K = 8 (two core matrices along K); step s starts at
//   base + s * 2 * LBO.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace esk {
namespace tc {

ESNMF_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// tile byte offset of element (r, k) in the K-major no-swizzle layout above
ESNMF_DEV uint32_t kmajor_off(int r, int k, int K) {
  return (uint32_t)((r >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

// 64-bit shared-memory matrix descriptor (SM100 UMMA, version 1, no swizzle)
ESNMF_DEV uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  // base_offset 0, lbo_mode 0, layout_type 0 (SWIZZLE_NONE)
  return d;
}

// 32-bit instruction descriptor: kind::tf32, fp32 accumulate, K-major A and B
ESNMF_DEV uint32_t make_idesc_tf32(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format F32
  d |= 2u << 7;                    // a_format TF32
  d |= 2u << 10;                   // b_format TF32
  d |= (uint32_t)(N >> 3) << 17;   // n_dim
  d |= (uint32_t)(M >> 4) << 24;   // m_dim
  return d;
}

// round-to-nearest tf32 value (low 13 bits zero) in an fp32 container
ESNMF_DEV float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ---- TMEM allocation (one full warp) ----
ESNMF_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
ESNMF_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

ESNMF_DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
ESNMF_DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// make generic-proxy shared-memory writes visible to the tensor core (async proxy)
ESNMF_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T (both K-major), issued by one thread
ESNMF_DEV void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// arrive on an mbarrier when all previously issued MMAs of this thread complete
ESNMF_DEV void mma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

ESNMF_DEV void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
ESNMF_DEV void mbar_wait(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

// the same wait, but the warp may be suspended in hardware (up to `ns`
// nanoseconds per try) until the phase completes instead of re-polling: waits
// that are not latency-critical no longer take issue slots from the other warps
// of their SM sub-partition (the head's epilogue spun ~220 times per tile)
ESNMF_DEV void mbar_wait_sleep(uint64_t* mbar, uint32_t phase, uint32_t ns) {
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAIT_%=;\n\t}" ::"r"(smem_u32(mbar)),
      "r"(phase), "r"(ns)
      : "memory");
}

// 8 consecutive fp32 columns of this thread's TMEM lane (warp w: lanes 32(w%4)..)
ESNMF_DEV void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}


// 32-bit instruction descriptor: kind::f16 with fp16 A and B, fp32 accumulate,
// K-major A and B (a_format = b_format = 0 = F16)
ESNMF_DEV uint32_t make_idesc_f16(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                    // c_format F32
  d |= (uint32_t)(N >> 3) << 17;   // n_dim
  d |= (uint32_t)(M >> 4) << 24;   // m_dim
  return d;
}

// D[tmem] (+)= A[smem] * B[smem]^T, fp16 inputs (K = 16 per instruction)
ESNMF_DEV void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// make mbarrier initialisation visible to the async proxy (bulk copies, MMA commits)
ESNMF_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

ESNMF_DEV void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}
ESNMF_DEV void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
}

// add to the transaction count of the current phase without arriving
ESNMF_DEV void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, no tensor map); completes `bytes`
// of the mbarrier's transaction count.  16-byte aligned, bytes % 16 == 0.
ESNMF_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mbar))
      : "memory");
}

// bulk prefetch of global memory into L2 (no completion mechanism)
ESNMF_DEV void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// 16 consecutive fp32 columns of this thread's TMEM lane (no wait: call tmem_wait_ld)
ESNMF_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
ESNMF_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte offset of element (r, k) of an R x K fp16 tile, K-major, no swizzle:
// 8-row x 16-byte core matrices, LBO = 128 (along K), SBO = (K / 8) * 128
ESNMF_DEV uint32_t kmajor_off16(int r, int k, int K) {
  return (uint32_t)((r >> 3) * (K / 8) * 128 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

}  // namespace tc
}  // namespace esk
