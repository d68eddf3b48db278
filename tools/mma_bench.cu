// mma_bench.cu -- tcgen05.mma throughput microbenchmark (cycles per MMA vs N, A from TMEM
// or SMEM, kind::tf32 / kind::f16), one CTA per SM, operands are garbage (timing only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"

using namespace hg;

__device__ __forceinline__ void mma_tf32_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc));
}

// warp-uniform issue: the whole warp runs the loop, one elected lane issues
__device__ __forceinline__ void mma_tf32_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p, e;\n\t"
                 "elect.sync _|e, 0xffffffff;\n\t"
                 "setp.ne.b32 p, 1, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc));
}

__global__ void k_bench(int mode, int N, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    if (mode >= 5 && threadIdx.x < 32) {
        const uint32_t sb = tc::smem_u32(smem);
        const uint64_t bdesc = tc::sdesc(sb, 4096, 128);
        const uint32_t idesc = tc::idesc_tf32(128, N);
        long long t0 = clock64();
        if (mode == 5) {
#pragma unroll 4
            for (int i = 0; i < iters; ++i) mma_tf32_ts_elect(t, t + 256, bdesc, idesc);
        } else {
#pragma unroll 4
            for (int i = 0; i < iters; ++i)
                mma_tf32_ts_elect(t + (i & 3) * 64, t + 256 + (i & 3) * 8, bdesc + (i & 3) * 32, idesc);
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) tc::mma_commit(&bar);
        __syncwarp();
        tc::mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    } else if (mode < 5 && threadIdx.x == 0) {
        const uint32_t sb = tc::smem_u32(smem);
        const uint64_t bdesc = tc::sdesc(sb, 4096, 128);
        const uint64_t adesc = tc::sdesc(sb + 65536, 4096, 128);
        uint32_t idesc = tc::idesc_tf32(128, N);
        if (mode == 2) idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);  // bf16
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (mode == 0) tc::mma_tf32_ts(t, t + 256, bdesc, idesc, 1);
            else if (mode == 3) tc::mma_tf32_ts(t + (i & 3) * 64, t + 256, bdesc, idesc, 1);
            else if (mode == 4) tc::mma_tf32_ts(t + (i & 1) * 128, t + 256, bdesc, idesc, 1);
            else if (mode == 1) mma_tf32_ss(t, adesc, bdesc, idesc);
            else mma_f16_ts(t, t + 256, bdesc, idesc);
        }
        long long t1 = clock64();
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(t, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"tf32 TS", "tf32 SS", "bf16 TS", "tf32 TS 4D", "tf32 TS 2D", "tf32 TS warp-elect", "tf32 TS warp-elect 4D"};
    for (int mode : {5, 6}) {
        for (int N : {16, 32, 48, 64, 96, 128}) {
            if (mode == 6 && N > 64) continue;
            int iters = 4096;
            k_bench<<<148, 128, 200 * 1024>>>(mode, N, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            double per = (double)h[1] / iters;
            double macs = 128.0 * N * (mode == 2 ? 16 : 8);
            printf("%s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma, %.0f MAC/cyc/SM %s\n",
                   names[mode], N, (double)h[0] / iters, per, macs / per,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
