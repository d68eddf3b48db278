// mbar_bench.cu -- latency of mbarrier operations as the engine uses them: try_wait on a
// phase that has already completed (with / without suspend hint), test_wait, arrive, and a
// tcgen05.st + wait::st round, each measured back to back in one warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__global__ void k(unsigned long long* out, int iters) {
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tb;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) tc::tmem_alloc(&tb, 512);
    __syncthreads();
    if (threadIdx.x == 0) tc::mbar_arrive(&bar[0]);   // phase 0 of bar[0] completes
    __syncthreads();
    tc::fence_after_sync();
    if (threadIdx.x < 32) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) tc::mbar_wait(&bar[0], 0);            // completed phase
        long long t1 = clock64();
        for (int i = 0; i < iters; ++i) tc::mbar_wait_spin(&bar[0], 0);
        long long t2 = clock64();
        for (int i = 0; i < iters; ++i) {                                    // arrive + wait own phase
            if (threadIdx.x == 0) tc::mbar_arrive(&bar[1]);
            __syncwarp();
            tc::mbar_wait(&bar[1], i & 1);
        }
        long long t3 = clock64();
        uint32_t r[16];
        for (int k = 0; k < 16; ++k) r[k] = k;
        for (int i = 0; i < iters; ++i) {
            tc::tmem_st16(tb + (i & 3) * 16, r);
            tc::wait_st();
        }
        long long t4 = clock64();
        for (int i = 0; i < iters; ++i) {
            tc::tmem_st16(tb + (i & 3) * 16, r);
            tc::tmem_st16(tb + 64 + (i & 3) * 16, r);
        }
        tc::wait_st();
        long long t5 = clock64();
        for (int i = 0; i < iters; ++i) {
            tc::fence_before_sync();
            __syncwarp();
            tc::fence_after_sync();
        }
        long long t6 = clock64();
        for (int i = 0; i < iters; ++i) {
            tc::tmem_st16(tb + (i & 3) * 16, r);
            tc::wait_st();
            tc::fence_before_sync();
            __syncwarp();
            if (threadIdx.x == 0) tc::mbar_arrive(&bar[1]);
            tc::mbar_wait(&bar[1], i & 1);
            tc::fence_after_sync();
        }
        long long t7 = clock64();
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
            out[5] = t6 - t5; out[6] = t7 - t6;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tb, 512);
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 128);
    const int iters = 1000;
    k<<<1, 128>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[7];
    cudaMemcpy(h, d, 56, cudaMemcpyDeviceToHost);
    printf("%s\n", cudaGetErrorString(e));
    printf("try_wait (done phase, suspend hint): %.1f cyc\n", h[0] / (double)iters);
    printf("test_wait spin (done phase):         %.1f cyc\n", h[1] / (double)iters);
    printf("arrive + wait (own phase):           %.1f cyc\n", h[2] / (double)iters);
    printf("tcgen05.st x16 + wait::st:           %.1f cyc\n", h[3] / (double)iters);
    printf("2 x tcgen05.st x16 (pipelined):      %.1f cyc\n", h[4] / (double)iters);
    printf("tcgen05.fence before/after + syncwarp: %.1f cyc\n", h[5] / (double)iters);
    printf("st + wait + fence + arrive + wait + fence: %.1f cyc\n", h[6] / (double)iters);
    return 0;
}
