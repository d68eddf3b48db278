// mbar_bench2.cu -- mbarrier try_wait throughput per SM: W warps of one CTA each poll an
// already-completed phase `iters` times (one lane or the whole warp issuing).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__global__ void k(unsigned long long* out, int iters, int nwarps) {
    __shared__ uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) tc::mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x < 16) tc::mbar_arrive(&bar[threadIdx.x]);
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    long long t0 = clock64();
    if (warp < nwarps)
        for (int i = 0; i < iters; ++i) tc::mbar_wait(&bar[(warp + i) & 15], 0);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    const int iters = 2000;
    for (int nw : {1, 2, 4, 8, 16}) {
        k<<<148, 512>>>(d, iters, nw);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%2d warps polling: %.1f cycles per wait per warp, %.1f cycles per wait per SM %s\n", nw,
               h / (double)iters, h / (double)iters / nw, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
