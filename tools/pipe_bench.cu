// pipe_bench.cu -- the tensor-core engine's per-entry pipeline, rebuilt from synthetic
// entries so each ingredient can be switched on separately and its cost per schedule entry
// measured (cycles / entry / SM, all 148 SMs busy).  Entry = 32 samples x 128 channels of
// values (16 KB), 4 in-reach blocks in 2 runs of 2 (weights 4 x 4 KB), 24 MMAs of N = 32.
//   F_MMA 1, F_STTM 2, F_VLDS 4, F_VCP 8, F_WCP 16, F_PROMO 32, F_SPIN 64
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "tc_bench_ptx.cuh"
using namespace hg;

enum { F_MMA = 1, F_STTM = 2, F_VLDS = 4, F_VCP = 8, F_WCP = 16, F_PROMO = 32, F_SPIN = 64, F_HALFN = 128 };
constexpr int NV = 3, NB = 4, NBF = 16, SEG = 16;
constexpr uint32_t VST = 16384, WST = 16384;

struct Smem {
    uint8_t W[NB][WST];
    uint8_t V[NV][VST];
    float M[128][196];
    uint64_t a_full[4], b_full[NB], v_full[NV], v_empty[NV], done[NBF], seg_done[2], seg_free[2];
    uint32_t tbase;
};

template <int F>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
    if (F & F_SPIN) tc::mbar_wait_spin(b, ph); else tc::mbar_wait(b, ph);
}

template <int F, int NA>
__global__ void __launch_bounds__(512, 1) k(const uint8_t* __restrict__ vsrc, const uint8_t* __restrict__ wsrc,
                                             size_t span, size_t vspan, uint32_t wbytes, int E, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem& s = *reinterpret_cast<Smem*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NAW = 8;   // A-producer warps
    if (warp == 0) tc::tmem_alloc(&s.tbase, 512);
    if (threadIdx.x == 32) {
        for (int i = 0; i < NA; ++i) tc::mbar_init(&s.a_full[i], NAW);
        for (int i = 0; i < NB; ++i) tc::mbar_init(&s.b_full[i], 1);
        for (int i = 0; i < NV; ++i) { tc::mbar_init(&s.v_full[i], 1); tc::mbar_init(&s.v_empty[i], NAW); }
        for (int i = 0; i < NBF; ++i) tc::mbar_init(&s.done[i], 1);
        for (int i = 0; i < 2; ++i) { tc::mbar_init(&s.seg_done[i], 1); tc::mbar_init(&s.seg_free[i], NAW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 128 * 196; i += 512) (&s.M[0][0])[i] = 0.f;
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = s.tbase;
    const long long t0 = clock64();
    const size_t cta_off = (size_t)blockIdx.x * 7919 * 256;
    if (warp == 0) {
        const uint32_t wb = tc::smem_u32(&s.W[0][0]);
        for (int c = 0; c < E; ++c) {
            const int seg = c / SEG, d = seg & 1;
            if ((F & F_PROMO) && c % SEG == 0 && seg >= 2) { wait<F>(&s.seg_free[d], ((seg >> 1) - 1) & 1); tc::fence_after_sync(); }
            wait<F>(&s.a_full[c % NA], (c / NA) & 1);
            wait<F>(&s.b_full[c % NB], (c / NB) & 1);
            tc::fence_after_sync();
            if (F & F_MMA) {
                const uint32_t b0 = wb + (c % NB) * WST;
                const uint32_t a0 = tm + 384 + (c % NA) * 64;
                const uint32_t db = tm + (F & F_PROMO ? d * 192 : 0);
                // run 1: blocks 0-1 (slots 0-1), run 2: blocks 4-5 (slots 2-3); hi at slot q, lo at +2 KB*4
                tc::mma12_3xtf32<2>(db + 0, a0, tc::sdesc_sw128_lo(b0), tc::sdesc_sw128_lo(b0 + 8192), tc::idesc_tf32(128, 32));
                tc::mma12_3xtf32<2>(db + 64, a0, tc::sdesc_sw128_lo(b0 + 4096), tc::sdesc_sw128_lo(b0 + 12288), tc::idesc_tf32(128, 32));
            }
            tc::mma_commit_warp(&s.done[c % NBF]);
            if ((F & F_PROMO) && (c % SEG == SEG - 1 || c == E - 1)) tc::mma_commit_warp(&s.seg_done[d]);
            __syncwarp();
        }
    } else if (warp == 1) {
        if (lane == 0)
            for (int c = 0; c < E; ++c) {
                const int sv = c % NV;
                if (c >= NV) wait<F>(&s.v_empty[sv], ((c / NV) - 1) & 1);
                if (F & F_VCP) {
                    tc::mbar_arrive_expect_tx(&s.v_full[sv], VST);
                    tc::bulk_g2s(&s.V[sv][0], vsrc + (cta_off + (size_t)c * VST) % vspan, VST, &s.v_full[sv]);
                } else {
                    tc::mbar_arrive(&s.v_full[sv]);
                }
            }
        __syncwarp();
    } else if (warp == 2) {
        if (lane == 0)
            for (int c = 0; c < E; ++c) {
                const int sb = c % NB;
                if (c >= NB) wait<F>(&s.done[(c - NB) % NBF], ((c - NB) / NBF) & 1);
                if (F & F_WCP) {
                    tc::mbar_arrive_expect_tx(&s.b_full[sb], wbytes);
                    tc::bulk_g2s(&s.W[sb][0], wsrc + (cta_off / 4 + (size_t)(c % 64) * WST) % span, wbytes, &s.b_full[sb]);
                } else {
                    tc::mbar_arrive(&s.b_full[sb]);
                }
            }
        __syncwarp();
    } else if (warp >= 4 && warp < 4 + NAW) {
        const int q4 = warp & 3, chl = q4 * 32 + lane, k0 = ((warp - 4) >> 2) * 16;
        uint32_t hi[16], lo[16];
        float acc = 0.f;
        uint32_t dmask = 0;
        for (int c = 0; c < E; ++c) {
            const int sv = c % NV;
            wait<F>(&s.v_full[sv], (c / NV) & 1);
            if (F & F_VLDS) {
                const float* vs = reinterpret_cast<const float*>(&s.V[sv][0]) + k0 * 128 + chl;
#pragma unroll
                for (int k = 0; k < 16; ++k) tc::split_tf32(vs[k * 128], hi[k], lo[k]);
                float t = 0.f;
#pragma unroll
                for (int k = 0; k < 16; ++k) t += __uint_as_float(lo[k]);
                acc += t;
                asm volatile("st.shared.u32 [%0], %1;" :: "r"(tc::smem_u32(&s.M[127][195])), "r"(__float_as_uint(t)) : "memory");
            } else {
#pragma unroll
                for (int k = 0; k < 16; ++k) { hi[k] = c + k; lo[k] = c - k; }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.v_empty[sv]);
            if (c >= NA) wait<F>(&s.done[(c - NA) % NBF], ((c - NA) / NBF) & 1);
            tc::fence_after_sync();
            if (F & F_STTM) {
                const uint32_t ta = tm + ((uint32_t)(q4 * 32) << 16) + 384 + (c % NA) * 64 + k0;
                tc::tmem_st16(ta, hi);
                tc::tmem_st16(ta + 32, lo);
                tc::wait_st();
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.a_full[c % NA]);
            if ((F & F_PROMO) && c >= SEG && c % SEG == NA) {
                const int sg = c / SEG - 1, d = sg & 1;
                wait<F>(&s.seg_done[d], (sg >> 1) & 1);
                tc::fence_after_sync();
                const int grp = (warp - 4) >> 2;
                for (int i = grp; i < 4; i += 2) {     // blocks 0, 1, 4, 5 touched in the segment
                    const int bb = (i & 1) + (i >> 1) * 4;
                    uint32_t r[16];
                    const uint32_t ta = tm + ((uint32_t)(q4 * 32) << 16) + d * 192 + (uint32_t)((bb % 12) * 16);
                    tc::tmem_ld16(ta, r);
                    tc::wait_ld();
                    uint32_t z[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) z[k] = 0u;
                    tc::tmem_st16(ta, z);
                    float* mr = &s.M[chl][(bb % 12) * 16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) mr[k] += __uint_as_float(r[k]);
                }
                tc::wait_st();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&s.seg_free[d]);
            }
        }
        dmask = __float_as_uint(acc);
        if (dmask == 0x7fffffffu) out[2] = dmask;
    }
    tc::fence_before_sync();
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(&out[0], (unsigned long long)(t1 - t0));
    if (warp == 0) tc::tmem_dealloc(tm, 512);
}

template <int F, int NA>
void run(const char* name, const uint8_t* v, const uint8_t* w, size_t span, unsigned long long* d, size_t vspan = (size_t)1 << 30, uint32_t wbytes = WST) {
    const int E = 4000, grid = 148;
    auto kern = k<F, NA>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem) + 1024);
    cudaMemset(d, 0, 24);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<grid, 512, sizeof(Smem) + 1024>>>(v, w, span, vspan, wbytes, E, d);   // warm
    cudaMemset(d, 0, 24);
    cudaEventRecord(e0);
    kern<<<grid, 512, sizeof(Smem) + 1024>>>(v, w, span, vspan, wbytes, E, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("%-34s vspan %5zu MB w %5u B NA=%d: %7.1f cycles/entry (clock64), %7.1f cycles/entry @1.965GHz (events) %s\n", name, vspan >> 20, wbytes, NA,
           h[0] / (double)grid / E, ms * 1e-3 * 1.965e9 / E, e == cudaSuccess ? "" : cudaGetErrorString(e));
}


// ---------------------------------------------------------------- v2 pipeline
// roles: W0 issuer, W1 V loader, W2 W loader, W4-7 A producers (32 samples / thread),
// W8-15 promoters: master sums in registers (group g = blocks 6g..6g+5, 96 floats / thread)
template <int NV2, int NB2>
struct Smem2 {
    uint8_t W[NB2][WST];
    uint8_t V[NV2][VST];
    uint64_t a_full[8], b_full[NB2], v_full[NV2], v_empty[NV2], done[NBF], seg_done[2], seg_free[2];
    uint32_t tbase;
};
template <int F, int NV2, int NB2, int NA>
__global__ void __launch_bounds__(512, 1) k2(const uint8_t* __restrict__ vsrc, const uint8_t* __restrict__ wsrc,
                                              size_t span, size_t vspan, uint32_t wbytes, int E, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    using SM = Smem2<NV2, NB2>;
    SM& s = *reinterpret_cast<SM*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NAW = 4, NPW = 8;
    constexpr uint32_t AC0 = 192;
    if (warp == 0) tc::tmem_alloc(&s.tbase, 512);
    if (threadIdx.x == 32) {
        for (int i = 0; i < NA; ++i) tc::mbar_init(&s.a_full[i], NAW);
        for (int i = 0; i < NB2; ++i) tc::mbar_init(&s.b_full[i], 1);
        for (int i = 0; i < NV2; ++i) { tc::mbar_init(&s.v_full[i], 1); tc::mbar_init(&s.v_empty[i], NAW); }
        for (int i = 0; i < NBF; ++i) tc::mbar_init(&s.done[i], 1);
        for (int i = 0; i < 2; ++i) { tc::mbar_init(&s.seg_done[i], 1); tc::mbar_init(&s.seg_free[i], NPW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = s.tbase;
    const long long t0 = clock64();
    const size_t cta_off = (size_t)blockIdx.x * 7919 * 256;
    if (warp == 0) {
        const uint32_t wb = tc::smem_u32(&s.W[0][0]);
        for (int c = 0; c < E; ++c) {
            const int seg = c / SEG, d = seg & 1;
            if ((F & F_PROMO) && c % SEG == 0 && seg >= 2) { wait<F>(&s.seg_free[d], ((seg >> 1) - 1) & 1); tc::fence_after_sync(); }
            wait<F>(&s.a_full[c % NA], (c / NA) & 1);
            wait<F>(&s.b_full[c % NB2], (c / NB2) & 1);
            tc::fence_after_sync();
            if (F & F_MMA) {
                const uint32_t b0 = wb + (c % NB2) * WST;
                const uint32_t a0 = tm + AC0 + (c % NA) * 64;
                const uint32_t db = tm + d * 96;
                const int nn = (F & F_HALFN) ? 16 : 32;
                tc::mma12_3xtf32<2>(db + 0, a0, tc::sdesc_sw128_lo(b0), tc::sdesc_sw128_lo(b0 + 8192), tc::idesc_tf32(128, nn));
                tc::mma12_3xtf32<2>(db + 64, a0, tc::sdesc_sw128_lo(b0 + 4096), tc::sdesc_sw128_lo(b0 + 12288), tc::idesc_tf32(128, nn));
            }
            tc::mma_commit_warp(&s.done[c % NBF]);
            if ((F & F_PROMO) && (c % SEG == SEG - 1 || c == E - 1)) tc::mma_commit_warp(&s.seg_done[d]);
            __syncwarp();
        }
    } else if (warp == 1) {
        if (lane == 0)
            for (int c = 0; c < E; ++c) {
                const int sv = c % NV2;
                if (c >= NV2) wait<F>(&s.v_empty[sv], ((c / NV2) - 1) & 1);
                if (F & F_VCP) {
                    tc::mbar_arrive_expect_tx(&s.v_full[sv], VST);
                    tc::bulk_g2s(&s.V[sv][0], vsrc + (cta_off + (size_t)c * VST) % vspan, VST, &s.v_full[sv]);
                } else {
                    tc::mbar_arrive(&s.v_full[sv]);
                }
            }
        __syncwarp();
    } else if (warp == 2) {
        if (lane == 0)
            for (int c = 0; c < E; ++c) {
                const int sb = c % NB2;
                if (c >= NB2) wait<F>(&s.done[(c - NB2) % NBF], ((c - NB2) / NBF) & 1);
                if (F & F_WCP) {
                    tc::mbar_arrive_expect_tx(&s.b_full[sb], wbytes);
                    tc::bulk_g2s(&s.W[sb][0], wsrc + (cta_off / 4 + (size_t)(c % 64) * WST) % span, wbytes, &s.b_full[sb]);
                } else {
                    tc::mbar_arrive(&s.b_full[sb]);
                }
            }
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        const int q4 = warp & 3, chl = q4 * 32 + lane;
        uint32_t hi[32], lo[32];
        float acc = 0.f;
        for (int c = 0; c < E; ++c) {
            const int sv = c % NV2;
            wait<F>(&s.v_full[sv], (c / NV2) & 1);
            if (F & F_VLDS) {
                const float* vs = reinterpret_cast<const float*>(&s.V[sv][0]) + chl;
#pragma unroll
                for (int k = 0; k < 32; ++k) tc::split_tf32(vs[k * 128], hi[k], lo[k]);
                float t = 0.f;
#pragma unroll
                for (int k = 0; k < 32; ++k) t += __uint_as_float(lo[k]);
                acc += t;
                asm volatile("st.shared.u32 [%0], %1;" :: "r"(tc::smem_u32(&s.tbase) + 4), "r"(__float_as_uint(t)) : "memory");
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k) { hi[k] = c + k; lo[k] = c - k; }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.v_empty[sv]);
            if (c >= NA) wait<F>(&s.done[(c - NA) % NBF], ((c - NA) / NBF) & 1);
            tc::fence_after_sync();
            if (F & F_STTM) {
                const uint32_t ta = tm + ((uint32_t)(q4 * 32) << 16) + AC0 + (c % NA) * 64;
                tc::tmem_st32(ta, hi);
                tc::tmem_st32(ta + 32, lo);
                tc::wait_st();
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.a_full[c % NA]);
        }
        if (__float_as_uint(acc) == 0x7fffffffu) out[2] = 1;
    } else if (warp >= 8) {
        const int q4 = warp & 3, g = (warp - 8) >> 2;
        float m[96];
#pragma unroll
        for (int k = 0; k < 96; ++k) m[k] = 0.f;
        const int nseg = (E + SEG - 1) / SEG;
        if (F & F_PROMO)
            for (int sg = 0; sg < nseg; ++sg) {
                const int d = sg & 1;
                wait<F>(&s.seg_done[d], (sg >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t mask = 0x33u;   // blocks 0, 1, 4, 5
#pragma unroll
                for (int bl = 0; bl < 6; ++bl) {
                    const int b = 6 * g + bl;
                    if ((mask >> b) & 1u) {
                        uint32_t r[16];
                        const uint32_t ta = tm + ((uint32_t)(q4 * 32) << 16) + d * 96 + (uint32_t)((b % 6) * 16);
                        tc::tmem_ld16(ta, r);
                        tc::wait_ld();
                        uint32_t z[16];
#pragma unroll
                        for (int k = 0; k < 16; ++k) z[k] = 0u;
                        tc::tmem_st16(ta, z);
#pragma unroll
                        for (int k = 0; k < 16; ++k) m[bl * 16 + k] += __uint_as_float(r[k]);
                    }
                }
                tc::wait_st();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&s.seg_free[d]);
            }
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 96; ++k) t += m[k];
        if (__float_as_uint(t) == 0x7fffffffu) out[2] = 2;
    }
    tc::fence_before_sync();
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(&out[0], (unsigned long long)(t1 - t0));
    if (warp == 0) tc::tmem_dealloc(tm, 512);
}

template <int F, int NV2, int NB2, int NA = 2>
void run2(const char* name, const uint8_t* v, const uint8_t* w, size_t span, unsigned long long* d, size_t vspan = (size_t)1 << 30, uint32_t wbytes = WST) {
    const int E = 4000, grid = 148;
    auto kern = k2<F, NV2, NB2, NA>;
    const int sm = sizeof(Smem2<NV2, NB2>) + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<grid, 512, sm>>>(v, w, span, vspan, wbytes, E, d);
    cudaMemset(d, 0, 24);
    cudaEventRecord(e0);
    kern<<<grid, 512, sm>>>(v, w, span, vspan, wbytes, E, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[3];
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("v2 %-31s vspan %5zu MB w %5u B NV=%d NB=%d NA=%d: %7.1f cycles/entry (clock64), %7.1f @1.965GHz (events) %s\n", name, vspan >> 20, wbytes,
           NV2, NB2, NA, h[0] / (double)grid / E, ms * 1e-3 * 1.965e9 / E, e == cudaSuccess ? "" : cudaGetErrorString(e));
}


// ---------------------------------------------------------------- V tile throughput: bulk vs 2D TMA box
#include <cuda.h>
__global__ void __launch_bounds__(128, 1) kv(const __grid_constant__ CUtensorMap tm, const uint8_t* __restrict__ src,
                                              int mode, int E, int rows_total, int ncb, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    constexpr int NS = 6;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + NS * VST);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) tc::mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        unsigned seed = blockIdx.x * 2654435761u;
        for (int c = 0; c < E; ++c) {
            const int s = c % NS;
            if (c >= NS) tc::mbar_wait(&full[s], ((c / NS) - 1) & 1);
            seed = seed * 1664525u + 1013904223u;
            const int row = (int)((seed >> 8) % (unsigned)(rows_total - 32));
            const int cb = (int)(blockIdx.x % ncb) * 128;
            tc::mbar_arrive_expect_tx(&full[s], VST);
            if (mode == 0) tc::tma_load_2d(raw + s * VST, &tm, cb, row, &full[s]);
            else tc::bulk_g2s(raw + s * VST, src + ((size_t)(blockIdx.x % ncb) * rows_total + row) * 512, VST, &full[s]);
        }
        for (int c = E; c < E + NS; ++c) { const int s = c % NS; tc::mbar_wait(&full[s], ((c / NS) - 1) & 1); }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&out[0], (unsigned long long)(clock64() - t0));
}
void run_v(int mode, const char* name, uint8_t* v, size_t span, unsigned long long* d) {
    using encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                   const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    const int C = 4096, rows = (int)(span / (C * 4));
    alignas(64) CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
    const cuuint32_t box[2] = {128, 32};
    const cuuint32_t es[2] = {1, 1};
    ((encode_fn)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, v, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int E = 3000, grid = 148, sm = 6 * VST + 64;
    cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    kv<<<grid, 128, sm>>>(tm, v, mode, E, mode == 0 ? rows : rows / 32 * 32, 32, d);
    cudaMemset(d, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kv<<<grid, 128, sm>>>(tm, v, mode, E, mode == 0 ? rows : rows / 32 * 32, 32, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %.1f cycles/tile, %.2f TB/s %s\n", name, ms * 1e-3 * 1.965e9 / E, 148.0 * E * VST / (ms * 1e-3) / 1e12,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}


// ---------------------------------------------------------------- k3: a half-size pipeline (256 threads,
// 96 KB SMEM, 256 TMEM columns) to test 2 CTAs per SM.  Roles: W0 issuer, W1 V loader, W2 W loader,
// W3 promoter (LDTM of the touched blocks every SEG entries), W4-7 A producers (32 samples / thread).
struct Smem3 {
    uint8_t W[3][WST];
    uint8_t V[3][VST];
    uint64_t a_full[2], b_full[3], v_full[3], v_empty[3], done[NBF], seg_done, seg_free;
    uint32_t tbase;
};
template <int F>
__global__ void __launch_bounds__(256) k3(const uint8_t* __restrict__ vsrc, const uint8_t* __restrict__ wsrc,
                                          size_t span, size_t vspan, uint32_t wbytes, int E, int tcols,
                                          unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t raw[];
    Smem3& s = *reinterpret_cast<Smem3*>(raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NA = 2, NV3 = 3, NB3 = 3;
    if (warp == 0) {
        if (tcols == 256) tc::tmem_alloc(&s.tbase, 256); else tc::tmem_alloc(&s.tbase, 512);
    }
    if (threadIdx.x == 32) {
        for (int i = 0; i < NA; ++i) tc::mbar_init(&s.a_full[i], 4);
        for (int i = 0; i < NB3; ++i) tc::mbar_init(&s.b_full[i], 1);
        for (int i = 0; i < NV3; ++i) { tc::mbar_init(&s.v_full[i], 1); tc::mbar_init(&s.v_empty[i], 4); }
        for (int i = 0; i < NBF; ++i) tc::mbar_init(&s.done[i], 1);
        tc::mbar_init(&s.seg_done, 1);
        tc::mbar_init(&s.seg_free, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = s.tbase;
    const long long t0 = clock64();
    const size_t cta_off = (size_t)blockIdx.x * 7919 * 256;
    if (warp == 0) {
        const uint32_t wb = tc::smem_u32(&s.W[0][0]);
        uint32_t gs = 0;
        for (int c = 0; c < E; ++c) {
            if (c % SEG == 0 && c > 0) { tc::mbar_wait(&s.seg_free, (gs - 1) & 1); tc::fence_after_sync(); }
            tc::mbar_wait(&s.a_full[c % NA], (c / NA) & 1);
            tc::mbar_wait(&s.b_full[c % NB3], (c / NB3) & 1);
            tc::fence_after_sync();
            if (F & F_MMA) {
                const uint32_t b0 = wb + (c % NB3) * WST;
                const uint32_t a0 = tm + 128 + (c % NA) * 64;
                tc::mma12_3xtf32<2>(tm + 0, a0, tc::sdesc_sw128_lo(b0), tc::sdesc_sw128_lo(b0 + 8192), tc::idesc_tf32(128, 32));
                tc::mma12_3xtf32<2>(tm + 64, a0, tc::sdesc_sw128_lo(b0 + 4096), tc::sdesc_sw128_lo(b0 + 12288), tc::idesc_tf32(128, 32));
            }
            tc::mma_commit_warp(&s.done[c % NBF]);
            if (c % SEG == SEG - 1 || c == E - 1) { tc::mma_commit_warp(&s.seg_done); ++gs; }
            __syncwarp();
        }
    } else if (warp == 1) {
        if (lane == 0)
            for (int c = 0; c < E; ++c) {
                const int sv = c % NV3;
                if (c >= NV3) tc::mbar_wait(&s.v_empty[sv], ((c / NV3) - 1) & 1);
                tc::mbar_arrive_expect_tx(&s.v_full[sv], VST);
                tc::bulk_g2s(&s.V[sv][0], vsrc + (cta_off + (size_t)c * VST) % vspan, VST, &s.v_full[sv]);
            }
    } else if (warp == 2) {
        if (lane == 0)
            for (int c = 0; c < E; ++c) {
                const int sb = c % NB3;
                if (c >= NB3) tc::mbar_wait(&s.done[(c - NB3) % NBF], ((c - NB3) / NBF) & 1);
                tc::mbar_arrive_expect_tx(&s.b_full[sb], wbytes);
                tc::bulk_g2s(&s.W[sb][0], wsrc + (cta_off / 4 + (size_t)(c % 64) * WST) % span, wbytes, &s.b_full[sb]);
            }
    } else if (warp == 3) {
        const int nseg = (E + SEG - 1) / SEG;
        float acc = 0.f;
        for (int sg = 0; sg < nseg; ++sg) {
            tc::mbar_wait(&s.seg_done, sg & 1);
            tc::fence_after_sync();
            for (int b = 0; b < 4; ++b) {     // lane quarter 3 only (one warp): enough to model the hand-off
                uint32_t r[16];
                tc::tmem_ld16(tm + ((uint32_t)(96) << 16) + (uint32_t)((b & 1) * 16 + (b >> 1) * 64), r);
                tc::wait_ld();
                for (int k = 0; k < 16; ++k) acc += __uint_as_float(r[k]);
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.seg_free);
        }
        if (__float_as_uint(acc) == 0x7fffffffu) out[2] = 3;
    } else {
        const int q4 = warp & 3, chl = q4 * 32 + lane;
        uint32_t hi[32], lo[32];
        float acc = 0.f;
        for (int c = 0; c < E; ++c) {
            const int sv = c % NV3;
            tc::mbar_wait(&s.v_full[sv], (c / NV3) & 1);
            const float* vs = reinterpret_cast<const float*>(&s.V[sv][0]) + chl;
#pragma unroll
            for (int k = 0; k < 32; ++k) tc::split_tf32(vs[k * 128], hi[k], lo[k]);
            float t = 0.f;
#pragma unroll
            for (int k = 0; k < 32; ++k) t += __uint_as_float(lo[k]);
            acc += t;
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.v_empty[sv]);
            if (c >= NA) tc::mbar_wait(&s.done[(c - NA) % NBF], ((c - NA) / NBF) & 1);
            tc::fence_after_sync();
            const uint32_t ta = tm + ((uint32_t)(q4 * 32) << 16) + 128 + (c % NA) * 64;
            tc::tmem_st32(ta, hi);
            tc::tmem_st32(ta + 32, lo);
            tc::wait_st();
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s.a_full[c % NA]);
        }
        if (__float_as_uint(acc) == 0x7fffffffu) out[2] = 1;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&out[0], (unsigned long long)(clock64() - t0));
    if (warp == 0) tc::tmem_dealloc(tm, tcols == 256 ? 256 : 512);
}
template <int F>
void run3(const char* name, int per_sm, const uint8_t* v, const uint8_t* w, size_t span, unsigned long long* d,
          size_t vspan, uint32_t wbytes = WST) {
    const int E = 3000, grid = 148 * per_sm;
    auto kern = k3<F>;
    const int sm = sizeof(Smem3) + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    const int tcols = per_sm == 2 ? 256 : 512;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<grid, 256, sm>>>(v, w, span, vspan, wbytes, E, tcols, d);
    cudaMemset(d, 0, 24);
    cudaEventRecord(e0);
    kern<<<grid, 256, sm>>>(v, w, span, vspan, wbytes, E, tcols, d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("k3 %-30s %d CTA/SM vspan %5zu MB: %7.1f cycles per entry per SM (events) %s\n", name, per_sm, vspan >> 20,
           ms * 1e-3 * 1.965e9 / (E * per_sm), e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    int idx = 0;
#define RUN(...) do { if (only < 0 || only == idx) __VA_ARGS__; ++idx; } while (0)
    const size_t span = (size_t)1 << 30;
    uint8_t *v, *w;
    unsigned long long* d;
    cudaMalloc(&v, span + VST);
    cudaMalloc(&w, span + WST);
    cudaMemset(v, 0, span + VST);
    cudaMemset(w, 0, span + WST);
    cudaMalloc(&d, 64);
    constexpr int ALL = F_MMA | F_STTM | F_VLDS | F_VCP | F_WCP | F_PROMO;
    const size_t S = 32u << 20;
    RUN((run3<F_MMA>("pipeline", 1, v, w, span, d, S)));
    RUN((run3<F_MMA>("pipeline", 2, v, w, span, d, S)));
    RUN((run3<F_MMA>("pipeline", 1, v, w, span, d, span)));
    RUN((run3<F_MMA>("pipeline", 2, v, w, span, d, span)));
    RUN((run2<ALL, 6, 6, 2>("all", v, w, span, d, S)));
    RUN((run2<ALL, 6, 6, 2>("all (V from HBM) w16K", v, w, span, d)));
    return 0;
}
