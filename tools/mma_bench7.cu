// mma_bench6.cu -- tcgen05.mma (kind::tf32, A in TMEM, B SW128 K-major) cost per MMA when every
// MMA reads a distinct B tile (rotating over `nb` tiles spread over shared memory) and one of
// 8 A stages, as in the engine, vs the same operands every time.  Operands precomputed.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__global__ void k(int n, int nb, int iters, int cm, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar, cb[2];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); tc::mbar_init(&cb[0], 1); tc::mbar_init(&cb[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    if (warp == 0) {
        const uint32_t base = tc::sdesc_sw128_lo(tc::smem_u32(smem));
        const uint32_t idesc = tc::idesc_tf32(128, n);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            // B tile i % nb: 2 KB apart (distinct rows); A stage i % 4 (64 columns each)
            const uint32_t b = base + (uint32_t)(((i % nb) * 2048) >> 4);
            tc::mma12_3xtf32<2, 32>(t, t + 256 + (uint32_t)((i & 3) * 64 % 256), b, b + 8, idesc);
            if (cm > 0 && i % cm == cm - 1) tc::mma_commit_warp(&cb[(i / cm) & 1]);
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
    for (int cm : {0, 1, 2, 4})
        for (int n : {16, 32, 64}) {
            const int iters = 256, nb = 32;
            k<<<148, 128, 200 * 1024>>>(n, nb, iters, cm, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const double per = h[1] / (12.0 * iters);
            printf("commit every %d x12 MMAs, B tiles %2d N=%3d: %.1f cyc/mma (issue %.1f), %.0f MAC/cyc %s\n", cm, nb, n, per,
                   h[0] / (12.0 * iters), 128.0 * n * 8 / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
