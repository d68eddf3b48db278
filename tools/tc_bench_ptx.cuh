// tc_bench_ptx.cuh -- the micro-benchmarks' PTX wrappers: the engine's own (tc_ptx.cuh) plus
// the variants the benchmarks use that the engine no longer does (single MMAs with a full
// descriptor, per-thread commit, generic descriptors).  Tool-only.
#pragma once
#include "../paper_2207_04584_b200/csrc/tc_ptx.cuh"

namespace hg {
namespace tc {

// Shared-memory matrix descriptor, no swizzle (canonical K-major interleaved layout:
// 8 rows x 16 B core matrices; LBO = byte distance between the two K core matrices of
// one MMA, SBO = byte distance between 8-row groups).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;                   // version (sm_100)
    return d;                                 // base offset 0, layout SWIZZLE_NONE (0)
}

// Shared-memory matrix descriptor, K-major with 128-byte swizzle: 8-row x 128-B atoms
// (1024-B aligned), SBO = 1024 B between 8-row groups, LBO unused (1).  Advancing along K
// inside the atom adds the byte offset (>> 4) to the start address.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                   // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;         // SBO
    d |= (uint64_t)1 << 46;                   // version (sm_100)
    d |= (uint64_t)2 << 61;                   // layout: SWIZZLE_128B
    return d;
}

// Arrives on `bar` when all previously issued MMAs of this thread have completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}

// ---- MMA ---------------------------------------------------------------------------
// D[tmem] (+)= A[tmem] * B[smem desc]^T, kind::tf32, cta_group::1.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
        "}\n" :: "r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// One run of the 3xTF32 product over a 32-sample chunk: 4 K-steps x (hi*hi, hi*lo, lo*hi),
// 12 MMAs behind a single elect.  A stage in TMEM: hi at columns a0 + 8 ks, lo at
// a0 + 32 + 8 ks; B descriptors: hi at b0 + ks * KS_STEP (16-B units), lo at + lo_off.
// The first MMA accumulates iff acc0 != 0, the other 11 always accumulate.
template <int KS_STEP>
__device__ __forceinline__ void mma_run_3xtf32(uint32_t d, uint32_t a0, uint64_t b0,
                                               uint64_t lo_off, uint32_t idesc, uint32_t acc0) {
#define HG_MMA_KS(ka, kl, bo)                                                              \
    "add.u32 ah, %1, " #ka ";\n\t"                                                         \
    "add.u32 al, %1, " #kl ";\n\t"                                                         \
    "add.s64 bh, %2, %" #bo ";\n\t"                                                        \
    "add.s64 bl, bh, %5;\n\t"                                                              \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %3, t;\n\t"                    \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %3, t;\n\t"                    \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %3, t;\n\t"
    asm volatile(
        "{\n\t"
        ".reg .pred e, p, t;\n\t"
        ".reg .b32 ah, al;\n\t"
        ".reg .b64 bh, bl;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.u32 t, 0, 0;\n\t"
        "add.s64 bl, %2, %5;\n\t"
        "add.u32 al, %1, 32;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], bl, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], %2, %3, t;\n\t"
        HG_MMA_KS(8, 40, 6) HG_MMA_KS(16, 48, 7) HG_MMA_KS(24, 56, 8)
        "}\n" :: "r"(d), "r"(a0), "l"(b0), "r"(idesc), "r"(acc0), "l"(lo_off),
        "n"(KS_STEP), "n"(2 * KS_STEP), "n"(3 * KS_STEP));
#undef HG_MMA_KS
}

}  // namespace tc
}  // namespace hg
