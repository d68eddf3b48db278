// mma_bench4.cu -- does the tcgen05.mma rate at small N depend on accumulator reuse?  12 MMAs
// (tf32, A in TMEM, B SW128 K-major) behind one elect, issued with D regions: all the same
// (dep=1), alternating between 2 (dep=2), 4 (dep=4) or 12 distinct regions.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

template <int NREG>
__device__ __forceinline__ void run12(uint32_t d, uint32_t dstride, uint32_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 d1, d2, d3;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "add.u32 d1, %0, %4;\n\t"
        "add.u32 d2, d1, %4;\n\t"
        "add.u32 d3, d2, %4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d1], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d2], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d3], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d1], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d2], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d3], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d1], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d2], [%1], %2, %3, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [d3], [%1], %2, %3, 1;\n\t"
        "}\n" :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(dstride) : "memory");
}
__global__ void k_bench(int n, int dstride, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    if (warp == 0) {
        const uint64_t bd = tc::sdesc_sw128(tc::smem_u32(smem));
        const uint32_t idesc = tc::idesc_tf32(128, n);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) run12<1>(t, dstride, t + 448, bd, idesc);
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
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int n : {16, 32, 64, 96})
        for (int ds : {0, 1}) {
            const int iters = 512, dstride = ds ? n : 0;
            if (4 * n > 448) continue;
            k_bench<<<148, 128, 64 * 1024>>>(n, dstride, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double per = h[1] / (12.0 * iters);
            printf("N=%3d D regions %s: issue %.1f, total %.1f cyc/mma, %.0f MAC/cyc %s\n", n, ds ? "4 rotating" : "1 (same)",
                   h[0] / (12.0 * iters), per, 128.0 * n * 8 / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
