// tf32_semantics.cu -- how does tcgen05.mma kind::tf32 read a 32-bit operand whose low 13
// mantissa bits are non-zero: truncation or round-to-nearest?  A (TMEM) = 1.0 in column 0 and
// 0 elsewhere, B (SMEM, K-major SW128) row n = {x_n, 0, ...}: D[:, n] = tf32(x_n).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

__global__ void k(const float* xs, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tbase;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tc::tmem_alloc(&tbase, 64);
    if (threadIdx.x == 32) { tc::mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    // B: 16 rows x 32 tf32 (one 128-B swizzle row each), K-major SW128: row r at r*128, k-quad j at (j ^ (r&7))*16
    uint32_t* b = reinterpret_cast<uint32_t*>(smem);
    for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) b[i] = 0;
    __syncthreads();
    if (threadIdx.x < 16) {
        const int r = threadIdx.x;
        b[r * 32 + ((0 ^ (r & 7)) * 4)] = __float_as_uint(xs[r]);   // k = 0
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t t = tbase;
    // A: lane m, column 0 = 1.0, columns 1..7 = 0 (K = 8)
    if (warp < 4) {
        uint32_t a[16];
        for (int i = 0; i < 16; ++i) a[i] = 0;
        a[0] = __float_as_uint(1.0f);
        tc::tmem_st16(t + ((uint32_t)(warp * 32) << 16) + 32, a);
        tc::wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) {
        const uint64_t bd = tc::sdesc_sw128(tc::smem_u32(smem));
        const uint32_t idesc = tc::idesc_tf32(128, 16);
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 0;\n\t}\n"
                     :: "r"(t), "r"(t + 32), "l"(bd), "r"(idesc) : "memory");
        tc::mma_commit_warp(&bar);
        tc::mbar_wait(&bar, 0);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) {
        uint32_t r[16];
        tc::tmem_ld16(t, r);
        tc::wait_ld();
        if (lane == 0) for (int n = 0; n < 16; ++n) out[n] = __uint_as_float(r[n]);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(t, 64);
}
int main() {
    float hx[16];
    for (int n = 0; n < 16; ++n) {
        uint32_t bits = 0x3F800000u | (0x1FFFu & (0x0FFFu + 0x0100u * n));   // 1.0 + low-bit patterns
        if (n == 15) bits = 0x3F801FFFu;                                    // all 13 low bits set
        if (n == 14) bits = 0x3F801000u;                                    // exactly half an ulp
        if (n == 13) bits = 0x3F803000u;                                    // odd tf32 mantissa + half
        memcpy(&hx[n], &bits, 4);
    }
    float *dx, *dout;
    cudaMalloc(&dx, 64);
    cudaMalloc(&dout, 64);
    cudaMemcpy(dx, hx, 64, cudaMemcpyHostToDevice);
    k<<<1, 128, 16 * 128 + 1024>>>(dx, dout);
    cudaError_t e = cudaDeviceSynchronize();
    float ho[16];
    cudaMemcpy(ho, dout, 64, cudaMemcpyDeviceToHost);
    int trunc_ok = 0, rn_ok = 0;
    for (int n = 0; n < 16; ++n) {
        uint32_t x, y;
        memcpy(&x, &hx[n], 4);
        memcpy(&y, &ho[n], 4);
        const uint32_t tr = x & 0xFFFFE000u, rn = (x + 0x1000u) & 0xFFFFE000u;
        trunc_ok += y == tr;
        rn_ok += y == rn;
        printf("x=%08x  D=%08x  trunc=%08x  rn(away)=%08x\n", x, y, tr, rn);
    }
    printf("%s: matches truncation %d/16, round-to-nearest %d/16\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e), trunc_ok, rn_ok);
    return 0;
}
