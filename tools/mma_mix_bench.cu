// mma_mix_bench.cu -- cost per schedule entry of the accumulate kernel's MMA stream:
// R runs per entry of either 12 kind::tf32 MMAs (3xTF32: hi*hi, hi*lo, lo*hi per K-step) or
// 8 MMAs (per K-step one kind::tf32 hi*hi + one kind::f16 (bf16) MMA whose K = 16 pairs the
// two correction terms), A in TMEM, B K-major SW128 in shared memory, one commit per entry.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_mix_bench tools/mma_mix_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2207_04584_b200/csrc/tc_ptx.cuh"
using namespace hg;

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// 4 K-steps: tf32 hi*hi (A cols a0 + 8ks, B bh + 2ks) then bf16 pair (A cols a0 + 32 + 8ks, B bl + 2ks)
__device__ __forceinline__ void mma8_mix(uint32_t d, uint32_t a0, uint32_t bh_lo, uint32_t bl_lo,
                                         uint32_t idt, uint32_t idb) {
#define KS(bh, bl, ah, al)                                                              \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+" #ah "], " #bh ", %4, 1;\n\t"      \
    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+" #al "], " #bl ", %5, 1;\n\t"
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        ".reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
        ".reg .b64 h0, h1, h2, h3, l0, l1, l2, l3;\n\t"
        "add.u32 x1, %2, 2;\n\t" "add.u32 x2, %2, 4;\n\t" "add.u32 x3, %2, 6;\n\t"
        "add.u32 y1, %3, 2;\n\t" "add.u32 y2, %3, 4;\n\t" "add.u32 y3, %3, 6;\n\t"
        "mov.b64 h0, {%2, %6};\n\t" "mov.b64 h1, {x1, %6};\n\t" "mov.b64 h2, {x2, %6};\n\t" "mov.b64 h3, {x3, %6};\n\t"
        "mov.b64 l0, {%3, %6};\n\t" "mov.b64 l1, {y1, %6};\n\t" "mov.b64 l2, {y2, %6};\n\t" "mov.b64 l3, {y3, %6};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        KS(h0, l0, 0, 32) KS(h1, l1, 8, 40) KS(h2, l2, 16, 48) KS(h3, l3, 24, 56)
        "}\n" :: "r"(d), "r"(a0), "r"(bh_lo), "r"(bl_lo), "r"(idt), "r"(idb), "n"(tc::kDescHiSw128) : "memory");
#undef KS
}

// 12 MMAs (3xTF32 over 4 K-steps) with A from shared memory (K-major SW128 tiles: hi at ah_lo,
// lo at al_lo), B as in mma12_3xtf32
__device__ __forceinline__ void mma12_ss(uint32_t d, uint32_t ah_lo, uint32_t al_lo, uint32_t bh_lo, uint32_t bl_lo,
                                         uint32_t idesc) {
#define KS(ah, al, bh, bl)                                                          \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], " #ah ", " #bh ", %5, 1;\n\t"     \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], " #ah ", " #bl ", %5, 1;\n\t"     \
    "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], " #al ", " #bh ", %5, 1;\n\t"
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        ".reg .b64 a0, a1, a2, a3, c0, c1, c2, c3, h0, h1, h2, h3, l0, l1, l2, l3;\n\t"
        ".reg .b32 t;\n\t"
        "mov.b64 a0, {%1, %6};\n\t" "add.u32 t, %1, 2;\n\t" "mov.b64 a1, {t, %6};\n\t" "add.u32 t, %1, 4;\n\t" "mov.b64 a2, {t, %6};\n\t" "add.u32 t, %1, 6;\n\t" "mov.b64 a3, {t, %6};\n\t"
        "mov.b64 c0, {%2, %6};\n\t" "add.u32 t, %2, 2;\n\t" "mov.b64 c1, {t, %6};\n\t" "add.u32 t, %2, 4;\n\t" "mov.b64 c2, {t, %6};\n\t" "add.u32 t, %2, 6;\n\t" "mov.b64 c3, {t, %6};\n\t"
        "mov.b64 h0, {%3, %6};\n\t" "add.u32 t, %3, 2;\n\t" "mov.b64 h1, {t, %6};\n\t" "add.u32 t, %3, 4;\n\t" "mov.b64 h2, {t, %6};\n\t" "add.u32 t, %3, 6;\n\t" "mov.b64 h3, {t, %6};\n\t"
        "mov.b64 l0, {%4, %6};\n\t" "add.u32 t, %4, 2;\n\t" "mov.b64 l1, {t, %6};\n\t" "add.u32 t, %4, 4;\n\t" "mov.b64 l2, {t, %6};\n\t" "add.u32 t, %4, 6;\n\t" "mov.b64 l3, {t, %6};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        KS(a0, c0, h0, l0) KS(a1, c1, h1, l1) KS(a2, c2, h2, l2) KS(a3, c3, h3, l3)
        "}\n" :: "r"(d), "r"(ah_lo), "r"(al_lo), "r"(bh_lo), "r"(bl_lo), "r"(idesc), "n"(tc::kDescHiSw128) : "memory");
#undef KS
}
// 12 identical MMAs (same D, A, B): the tensor core's own rate for this shape
__device__ __forceinline__ void mma12_same(uint32_t d, uint32_t a0, uint32_t bh_lo, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b64 h;\n\t"
        "mov.b64 h, {%2, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], h, %3, 1;\n\t}\n"
        :: "r"(d), "r"(a0), "r"(bh_lo), "r"(idesc), "n"(tc::kDescHiSw128) : "memory");
}

// mixed, grouped by kind: the 4 tf32 MMAs, then the 4 bf16 MMAs
__device__ __forceinline__ void mma8_grp(uint32_t d, uint32_t a0, uint32_t bh_lo, uint32_t bl_lo,
                                         uint32_t idt, uint32_t idb) {
    asm volatile(
        "{\n\t"
        ".reg .pred e;\n\t"
        ".reg .b32 x1, x2, x3, y1, y2, y3;\n\t"
        ".reg .b64 h0, h1, h2, h3, l0, l1, l2, l3;\n\t"
        "add.u32 x1, %2, 2;\n\t" "add.u32 x2, %2, 4;\n\t" "add.u32 x3, %2, 6;\n\t"
        "add.u32 y1, %3, 2;\n\t" "add.u32 y2, %3, 4;\n\t" "add.u32 y3, %3, 6;\n\t"
        "mov.b64 h0, {%2, %6};\n\t" "mov.b64 h1, {x1, %6};\n\t" "mov.b64 h2, {x2, %6};\n\t" "mov.b64 h3, {x3, %6};\n\t"
        "mov.b64 l0, {%3, %6};\n\t" "mov.b64 l1, {y1, %6};\n\t" "mov.b64 l2, {y2, %6};\n\t" "mov.b64 l3, {y3, %6};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+0], h0, %4, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+8], h1, %4, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+16], h2, %4, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+24], h3, %4, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+32], l0, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+40], l1, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+48], l2, %5, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+56], l3, %5, 1;\n\t"
        "}\n" :: "r"(d), "r"(a0), "r"(bh_lo), "r"(bl_lo), "r"(idt), "r"(idb), "n"(tc::kDescHiSw128) : "memory");
}

// one MMA (issued by the calling thread)
__device__ __forceinline__ void mma1(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc) {
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc) : "memory");
}
// 12 x R MMAs with the R runs interleaved per (K-step, product): consecutive MMAs hit different D
template <int R>
__device__ __forceinline__ void mma_interleaved(const uint32_t (&d)[R], uint32_t a0, const uint32_t (&b)[R], uint32_t idesc) {
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t a = a0 + (p == 2 ? 32 : 0) + 8 * ks;
                const uint32_t blo = b[r] + (p == 1 ? 128 : 0) + 2 * ks;
                const uint64_t desc = ((uint64_t)tc::kDescHiSw128 << 32) | blo;
                mma1(d[r], a, desc, idesc);
            }
}

__global__ void k(int mode, int n, int runs, int entries, int commit, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar, cb[16];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 32) {
        tc::mbar_init(&bar, 1);
        for (int i = 0; i < 16; ++i) tc::mbar_init(&cb[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    if (warp == 0) {
        const uint32_t base = tc::sdesc_sw128_lo(tc::smem_u32(smem));
        const uint32_t idt = tc::idesc_tf32(128, n), idb = idesc_bf16(128, n);
        long long t0 = clock64();
        for (int i = 0; i < entries; ++i) {
            if (mode >= 2) {
                const uint32_t a0 = t + 384 + (uint32_t)((i & 1) * 64);
                if (threadIdx.x == 0) {
                    if (runs == 2) {
                        uint32_t dd[2], bb[2];
                        for (int r = 0; r < 2; ++r) { bb[r] = base + (uint32_t)((((i * 2 + r) % 24) * 4096) >> 4); dd[r] = t + (uint32_t)(r * 48); }
                        mma_interleaved<2>(dd, a0, bb, idt);
                    } else {
                        uint32_t dd[4], bb[4];
                        for (int r = 0; r < 4; ++r) { bb[r] = base + (uint32_t)((((i * 4 + r) % 24) * 4096) >> 4); dd[r] = t + (uint32_t)(r * 80); }
                        mma_interleaved<4>(dd, a0, bb, idt);
                    }
                }
                __syncwarp();
            } else
            for (int r = 0; r < runs; ++r) {
                // B slot (i * runs + r) % 24 of 4 KB (hi 2 KB then lo), D at column 48 r % 384
                const uint32_t b = base + (uint32_t)((((i * runs + r) % 24) * 4096) >> 4);
                const uint32_t d = t + (uint32_t)((r * 48) % 336);
                const uint32_t a0 = t + 384 + (uint32_t)((i & 1) * 64);
                if (mode == 0) tc::mma12_3xtf32<2, 32>(d, a0, b, b + 128, idt);
                else if (mode == 1) mma8_mix(d, a0, b, b + 128, idt, idb);
                else if (mode == 4) {
                    // A tiles at 100 KB (hi) and 116 KB (lo), 16 KB each (128 rows x 128 B)
                    const uint32_t ah = tc::sdesc_sw128_lo(tc::smem_u32(smem + 102400 + (i & 1) * 32768));
                    mma12_ss(d, ah, ah + 1024, b, b + 128, idt);
                } else if (mode == 6) mma8_grp(d, a0, b, b + 128, idt, idb);
                else mma12_same(d, a0, b, idt);
            }
            if (commit) tc::mma_commit_warp(&cb[i & 15]);
        }
        long long t1 = clock64();
        tc::mma_commit_warp(&bar);
        tc::mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(t, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int commit : {1})
        for (int mode : {0, 1, 6})
            for (int n : {16, 32, 48, 64, 96, 128, 192}) {
                const int runs = mode == 3 ? 4 : (n >= 96 ? 1 : 2), entries = 512;
                if (mode == 4) {   // B slots must stay below the A tiles: 24 x 4 KB = 96 KB ok
                }
                k<<<148, 128, 200 * 1024>>>(mode, n, runs, entries, commit, d);
                cudaError_t e = cudaDeviceSynchronize();
                unsigned long long h[2] = {0, 0};
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                const int per_run = (mode == 1 || mode == 6) ? 8 : 12;
                const double per_entry = (double)h[1] / entries, per_mma = per_entry / (runs * per_run);
                printf("commit %d %s N=%3d: %7.1f cyc/entry (%d runs), %5.1f cyc/MMA, floor %5.1f, %s\n", commit,
                       mode == 0 ? "3xTF32 12/run" : mode == 1 ? "mixed   8/run" : mode == 2 ? "3xTF32 ilv x2" : mode == 3 ? "3xTF32 ilv x4" : mode == 4 ? "3xTF32 SS-A  " : mode == 6 ? "mixed grouped" : "same MMA x12 ", n, per_entry, runs, per_mma, 128.0 * n / 256,
                       e == cudaSuccess ? "ok" : cudaGetErrorString(e));
            }
    return 0;
}
