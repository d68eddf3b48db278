// a_bench.cu -- cycles per chunk of the A-producer path (LDS 32 values, tf32 split,
// 2 x tcgen05.st.32x32b.x32, wait::st) for 4 warps, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__global__ void k(int mode, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    float* V = reinterpret_cast<float*>(smem);
    for (int i = threadIdx.x; i < 5 * 4096; i += blockDim.x) V[i] = i * 0.001f;
    __syncthreads();
    long long t0 = clock64();
    uint32_t acc = 0;
    const int chl = (warp & 3) * 32 + lane;
    for (int c = 0; c < iters; ++c) {
        uint32_t hi[32], lo[32];
        const float* vs = V + (c % 5) * 4096 + chl;
        if (mode >= 3) {
#pragma unroll
            for (int k = 0; k < 32; ++k) { hi[k] = c + k; lo[k] = c - k; }
        } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) tc::split_tf32(vs[k * 128], hi[k], lo[k]);
        }
        if (mode >= 1) {
            const uint32_t ta = t + ((uint32_t)((warp & 3) * 32) << 16) + 256 + (c & 3) * 64;
            tc::tmem_st32(ta, hi);
            tc::tmem_st32(ta + 32, lo);
            if (mode == 2 || mode == 4) tc::wait_st();
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += hi[k] ^ lo[k];
        }
    }
    tc::wait_st();
    long long t1 = clock64();
    if (blockIdx.x == 0 && lane == 0) out[warp] = t1 - t0;
    if (acc == 12345) out[8] = acc;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(t, 512);
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 128);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int mode : {0, 1, 2, 3, 4}) {
        int iters = 2000;
        k<<<148, 128, 90 * 1024>>>(mode, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("mode %d (0 split, 1 +st, 2 +wait::st, 3 st only, 4 st+wait): %.1f cycles/chunk %s\n", mode, (double)h[0] / iters, e ? cudaGetErrorString(e) : "");
    }
}
