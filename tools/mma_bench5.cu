// mma_bench4.cu -- does the tcgen05.mma rate at small N depend on accumulator reuse?  12 MMAs
// (tf32, A in TMEM, B SW128 K-major) behind one elect, issued with D regions: all the same
// (dep=1), alternating between 2 (dep=2), 4 (dep=4) or 12 distinct regions.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__device__ __forceinline__ void run12(uint32_t d, uint32_t a1, uint32_t a2, uint32_t a3, uint64_t b1, uint64_t b2, uint64_t b3, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %5, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %6, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %6, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %4, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %5, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %6, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %6, %7, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %4, %7, 1;\n\t"
        "}\n" :: "r"(d), "r"(a1), "r"(a2), "r"(a3), "l"(b1), "l"(b2), "l"(b3), "r"(idesc) : "memory");
}
__global__ void k_bench(int n, int mode, int iters, unsigned long long* out) {
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
        const uint32_t a1 = t + 448, a2 = (mode & 1) ? t + 456 : a1, a3 = (mode & 1) ? t + 464 : a1;
        const uint64_t b1 = bd, b2 = (mode & 2) ? bd + 2 : bd, b3 = (mode & 2) ? bd + 1024 : bd;
        for (int i = 0; i < iters; ++i) run12(t, a1, a2, a3, b1, b2, b3, idesc);
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
        for (int ds : {0, 1, 2, 3}) {
            const int iters = 512;
            k_bench<<<148, 128, 64 * 1024>>>(n, ds, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double per = h[1] / (12.0 * iters);
            printf("N=%3d vary A %d B %d: issue %.1f, total %.1f cyc/mma, %.0f MAC/cyc %s\n", n, ds & 1, ds >> 1,
                   h[0] / (12.0 * iters), per, 128.0 * n * 8 / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
