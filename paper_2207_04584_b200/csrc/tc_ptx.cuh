// tc_ptx.cuh -- thin inline-PTX wrappers for the sm_100a features the tensor-core engine
// uses: TMEM allocation, tcgen05.mma (kind::tf32, A from TMEM), tcgen05.ld/st,
// tcgen05.commit -> mbarrier, and the async-proxy fences.
#pragma once

#include <stdint.h>

namespace hg {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// ---- TMEM allocation (one warp) ---------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(dst_smem)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols));
}

// ---- fences ------------------------------------------------------------------------
__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- mbarrier ----------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
// Wait for the phase with the given parity to complete.  try_wait with a suspend-time hint
// parks the warp in hardware until the phase flips (or the hint expires) instead of
// spinning on the issue slots the producer warps need.
#ifndef HG_MBAR_SUSPEND_NS
#define HG_MBAR_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if defined(HG_MBAR_SPIN)
    // spin on the non-blocking test (no suspension: lowest wake-up latency)
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
#elif defined(HG_MBAR_NOHINT)
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
#else
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" :: "r"(smem_u32(bar)), "r"(parity), "n"(HG_MBAR_SUSPEND_NS) : "memory");
#endif
}
// Spin on the non-blocking test: for the single-warp roles on the critical hand-off chain
// (MMA issuers, loaders), where wake-up latency matters more than the issue slots
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t"
        "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Bulk async copy global -> shared (contiguous bytes, 16-B aligned, multiple of 16),
// completion signalled as tx bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// 2D tensor-map (TMA) load of one box into shared memory; coordinates innermost first.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        :: "r"(smem_u32(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];"
                 :: "l"(tmap), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(src), "r"(bytes) : "memory");
}

// ---- MMA ---------------------------------------------------------------------------
// The same 12 MMAs issued so that ptxas keeps the operand arithmetic in uniform registers:
// TMEM operands as [base + immediate] (A hi at a0 + 8 ks, lo at a0 + 32 + 8 ks) and the B
// descriptors built inside the asm from their low words (start address, LBO) with the
// constant high word of a K-major SWIZZLE_128B descriptor (SBO = 1024 B, version 1), the
// K-step advancing the start address by KS_STEP (16-B units).  Each base value is moved to a
// uniform register once per run instead of once per MMA.
constexpr uint32_t kDescHiSw128 = 0x40004040u;   // layout 2 << 61 | version << 46 | (1024 >> 4) << 32
template <int KS_STEP, int ALO = 32>
__device__ __forceinline__ void mma12_3xtf32(uint32_t d, uint32_t a0, uint32_t bh_lo, uint32_t bl_lo,
                                             uint32_t idesc) {
#define HG_MMA12_KS(bh, bl, ah, al)                                                      \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+" #ah "], " #bh ", %4, 1;\n\t"       \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+" #ah "], " #bl ", %4, 1;\n\t"       \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+" #al "], " #bh ", %4, 1;\n\t"
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        ".reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
        ".reg .b64 h0, h1, h2, h3, l0, l1, l2, l3;\n\t"
        "add.u32 x1, %2, %5;\n\t"
        "add.u32 x2, %2, %6;\n\t"
        "add.u32 x3, %2, %7;\n\t"
        "add.u32 y1, %3, %5;\n\t"
        "add.u32 y2, %3, %6;\n\t"
        "add.u32 y3, %3, %7;\n\t"
        "mov.b64 h0, {%2, %8};\n\t"
        "mov.b64 h1, {x1, %8};\n\t"
        "mov.b64 h2, {x2, %8};\n\t"
        "mov.b64 h3, {x3, %8};\n\t"
        "mov.b64 l0, {%3, %8};\n\t"
        "mov.b64 l1, {y1, %8};\n\t"
        "mov.b64 l2, {y2, %8};\n\t"
        "mov.b64 l3, {y3, %8};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        HG_MMA12_KS(h0, l0, 0, %9) HG_MMA12_KS(h1, l1, 8, %10)
        HG_MMA12_KS(h2, l2, 16, %11) HG_MMA12_KS(h3, l3, 24, %12)
        "}\n" :: "r"(d), "r"(a0), "r"(bh_lo), "r"(bl_lo), "r"(idesc), "n"(KS_STEP),
        "n"(2 * KS_STEP), "n"(3 * KS_STEP), "n"(kDescHiSw128), "n"(ALO), "n"(ALO + 8),
        "n"(ALO + 16), "n"(ALO + 24) : "memory");
#undef HG_MMA12_KS
}
// Mixed-precision variant (span layout of the precomputed weight image): per K-step one
// kind::tf32 MMA of the hi parts (A cols a0 + 8 ks, B at bh) and one kind::f16 (bf16) MMA of
// K = 16 that pairs the two correction terms (A cols a0 + ALO + 8 ks hold {bf16(v), bf16(v_lo)}
// per sample, B at bl holds {bf16(w_lo), bf16(w_hi)}): 8 MMAs instead of 12.
template <int KS_STEP, int ALO = 32>
__device__ __forceinline__ void mma8_mix(uint32_t d, uint32_t a0, uint32_t bh_lo, uint32_t bl_lo,
                                         uint32_t idt, uint32_t idb) {
#define HG_MMA8_KS(bh, bl, ah, al)                                                       \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+" #ah "], " #bh ", %4, 1;\n\t"       \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+" #al "], " #bl ", %5, 1;\n\t"
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        ".reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
        ".reg .b64 h0, h1, h2, h3, l0, l1, l2, l3;\n\t"
        "add.u32 x1, %2, %6;\n\t"
        "add.u32 x2, %2, %7;\n\t"
        "add.u32 x3, %2, %8;\n\t"
        "add.u32 y1, %3, %6;\n\t"
        "add.u32 y2, %3, %7;\n\t"
        "add.u32 y3, %3, %8;\n\t"
        "mov.b64 h0, {%2, %9};\n\t"
        "mov.b64 h1, {x1, %9};\n\t"
        "mov.b64 h2, {x2, %9};\n\t"
        "mov.b64 h3, {x3, %9};\n\t"
        "mov.b64 l0, {%3, %9};\n\t"
        "mov.b64 l1, {y1, %9};\n\t"
        "mov.b64 l2, {y2, %9};\n\t"
        "mov.b64 l3, {y3, %9};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        HG_MMA8_KS(h0, l0, 0, %10) HG_MMA8_KS(h1, l1, 8, %11)
        HG_MMA8_KS(h2, l2, 16, %12) HG_MMA8_KS(h3, l3, 24, %13)
        "}\n" :: "r"(d), "r"(a0), "r"(bh_lo), "r"(bl_lo), "r"(idt), "r"(idb), "n"(KS_STEP),
        "n"(2 * KS_STEP), "n"(3 * KS_STEP), "n"(kDescHiSw128), "n"(ALO), "n"(ALO + 8),
        "n"(ALO + 16), "n"(ALO + 24) : "memory");
#undef HG_MMA8_KS
}
// low word of a K-major SWIZZLE_128B descriptor (start address >> 4, LBO field 1)
__device__ __forceinline__ uint32_t sdesc_sw128_lo(uint32_t saddr) {
    return ((saddr >> 4) & 0x3FFFu) | (1u << 16);
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
        "}\n" :: "r"(smem_u32(bar)) : "memory");
}
// Instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)                          // c_format = F32
         | (2u << 7)                          // a_format = TF32
         | (2u << 10)                         // b_format = TF32
         | ((uint32_t)(N >> 3) << 17)         // n_dim
         | ((uint32_t)(M >> 4) << 24);        // m_dim
}

// Instruction descriptor: kind::f16 with bf16 A/B (K-major), D fp32, M x N.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4)                          // c_format = F32
         | (1u << 7)                          // a_format = BF16
         | (1u << 10)                         // b_format = BF16
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}
// {bf16(x) in the low half, bf16(y) in the high half}, round to nearest even
__device__ __forceinline__ uint32_t pack_bf16(float x, float y) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(y), "f"(x));
    return r;
}

// ---- TMEM <-> registers (32 lanes x 32 bit, per warp) ------------------------------
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, "
        "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, "
        "%27, %28, %29, %30, %31, %32};"
        :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
           "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
           "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]),
           "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
           "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}
__device__ __forceinline__ void tmem_st32p(uint32_t taddr, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, "
        "%10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, "
        "%27, %28, %29, %30, %31, %32};"
        :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
           "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
           "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]),
           "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
           "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, "
        "%10, %11, %12, %13, %14, %15, %16};"
        :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
           "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
           "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
        "%10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr) : "memory");
}

// x = hi + lo with hi = x rounded to tf32 (nearest, ties away from zero, on the bit
// pattern) and lo = x - hi exact in fp32 (|lo| <= 2^-11 |x|); the tensor core reads lo's
// top 19 bits, so hi + lo carries ~21 significant bits of x.
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

}  // namespace tc
}  // namespace hg
