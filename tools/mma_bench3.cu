// mma_bench3.cu -- per-instruction cost of tcgen05.mma vs N for operand sources / kinds:
// TS tf32 (A in TMEM), SS tf32 (A in SMEM, MN-major SW128), TS f16 (K = 16).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__device__ __forceinline__ uint64_t sdesc_mn128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__global__ void k_bench(int mode, int n, int iters, unsigned long long* out) {
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
        const uint64_t ad = sdesc_mn128(tc::smem_u32(smem + 65536), 4096, 1024);
        uint32_t idesc = tc::idesc_tf32(128, n);
        if (mode == 1) idesc |= 1u << 15;                 // A MN-major
        if (mode == 2) idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);  // f16 in, f32 acc
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (mode == 2) {
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t}"
                             :: "r"(t), "r"(t + 256 + (i & 3) * 8), "l"(bd + (i & 3) * 2), "r"(idesc) : "memory");
            } else if (mode == 0) {
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n\t}"
                             :: "r"(t), "r"(t + 256 + (i & 3) * 8), "l"(bd + (i & 3) * 2), "r"(idesc) : "memory");
            } else {
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n\t}"
                             :: "r"(t), "l"(ad + (i & 3) * 64), "l"(bd + (i & 3) * 2), "r"(idesc) : "memory");
            }
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
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"TS tf32", "SS tf32 A-MN", "TS f16"};
    for (int mode : {0, 1, 2})
        for (int n : {16, 32, 64, 96, 128, 192, 256}) {
            int iters = 2048;
            k_bench<<<148, 128, 200 * 1024>>>(mode, n, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const int K = mode == 2 ? 16 : 8;
            printf("%-13s N=%3d: %.1f cyc/mma, %.0f MAC/cyc %s\n", names[mode], n, h[1] / (double)iters,
                   128.0 * n * K / (h[1] / (double)iters), e == cudaSuccess ? "" : cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
        }
    return 0;
}
