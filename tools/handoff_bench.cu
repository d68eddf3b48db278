// handoff_bench.cu -- latency of a hand-off between two warps of one CTA: ping-pong through
// two mbarriers (try_wait with suspend hint, or test_wait spinning) and through a named
// barrier (bar.sync with 64 threads), per one-way hand-off.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__global__ void k(int mode, int iters, unsigned long long* out) {
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    if (mode < 2) {
        for (int i = 0; i < iters; ++i) {
            if (warp == 0) {
                if (lane == 0) tc::mbar_arrive(&bar[0]);
                if (mode == 0) tc::mbar_wait(&bar[1], i & 1); else tc::mbar_wait_spin(&bar[1], i & 1);
            } else if (warp == 1) {
                if (mode == 0) tc::mbar_wait(&bar[0], i & 1); else tc::mbar_wait_spin(&bar[0], i & 1);
                if (lane == 0) tc::mbar_arrive(&bar[1]);
            }
        }
    } else {
        for (int i = 0; i < iters; ++i) {
            if (warp < 2) asm volatile("bar.sync 1, 64;" ::: "memory");
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const char* names[] = {"mbarrier try_wait (suspend)", "mbarrier test_wait (spin)", "named barrier bar.sync"};
    for (int mode = 0; mode < 3; ++mode) {
        const int iters = 2000;
        k<<<148, 128>>>(mode, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("%-30s: %.1f cycles per one-way hand-off %s\n", names[mode],
               h / (double)iters / (mode < 2 ? 2.0 : 1.0), e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
