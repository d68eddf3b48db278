// mma_bench2.cu -- cycles per tcgen05.mma (kind::tf32, A from TMEM, B K-major SW128) for the
// engine's issue pattern: runs of 12 MMAs (4 K-steps x 3 products) behind one elect, N = 16 r.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench2 mma_bench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"

using namespace hg;

__global__ void k_bench(int r, int runs_per_chunk, int chunks, int st_interfere, int commits, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar, cb[4];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) tc::mbar_init(&cb[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    if (warp == 0) {
        const uint64_t d0 = tc::sdesc_sw128(tc::smem_u32(smem));
        const uint32_t idesc = tc::idesc_tf32(128, 16 * r);
        long long t0 = clock64();
        for (int c = 0; c < chunks; ++c) {
            const uint32_t a0 = t + 256 + (c & 3) * 64;
            for (int k = 0; k < runs_per_chunk; ++k)
                tc::mma12_3xtf32<2>(t + (uint32_t)(k * 16 * r) % 64u, a0, d0 + (uint64_t)(k * r * 128), d0 + 1024 + (uint64_t)(k * r * 128), idesc);
            for (int k = 0; k < commits; ++k) tc::mma_commit_warp(&cb[k]);
        }
        long long t1 = clock64();
        tc::mma_commit_warp(&bar);
        tc::mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    } else if (warp >= 4 && warp < 8 && st_interfere) {
        uint32_t z[32];
        for (int k = 0; k < 32; ++k) z[k] = k;
        for (int c = 0; c < chunks * st_interfere; ++c) {
            tc::tmem_st32(t + ((uint32_t)((warp & 3) * 32) << 16) + 256 + ((c + 2) & 3) * 64, z);
            tc::wait_st();
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(t, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int cm : {0, 1}) {
        for (int r : {1, 2, 3, 4, 6, 8, 12}) {
            int chunks = 256, rpc = 2, st = 0;
            k_bench<<<148, 256, 64 * 1024>>>(r, rpc, chunks, st, cm, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            double n = (double)chunks * rpc * 12;
            printf("commits=%d r=%d N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma, %.0f MAC/cyc %s\n", cm, r, 16 * r,
                   h[0] / n, h[1] / n, 128.0 * 16 * r * 8 / (h[1] / n), e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
