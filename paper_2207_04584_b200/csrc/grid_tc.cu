// grid_tc.cu -- accumulate + normalise on the 5th-gen tensor cores (tcgen05, kind::tf32),
// error-compensated 3xTF32 so the sums keep fp32 accuracy.
//
// The contraction (Eq. 1 numerator): S[c][cell] = sum_n v[c][n] w(cell,n).
// Blocked: for a chunk of K = 32 plan-ordered candidate samples of one bin row and a
// 4x4-cell block,
//     D_block[128 ch][16 cells] += A[128 ch][32 samples] * B[16 cells][32 samples]^T
// with A = the chunk's values (channels on TMEM lanes), B = the (cell, sample) weights
// computed by the CTA's SIMT warps (each weight once per CTA, shared by its 128 channels:
// the paper's component-share principle), D = fp32 accumulators in TMEM.
// Each operand is split x = hi + lo with hi = tf32(x), lo = tf32(x - hi); three MMAs
// (hi*hi + hi*lo + lo*hi) reproduce the fp32 product to ~2^-22.
//
// CTA = 16x16 cells (16 blocks) x 128 channels, 512 threads, warp-specialised, all roles
// walking the same deterministic chunk sequence (bin rows of the tile's reach, 32-sample
// chunks, skipping chunks that reach no block):
//   warp 0 (lane 0) : MMA issuer.  Waits A-full and B-full of a stage, issues 12 MMAs per
//                     in-reach block, commits to the A-empty and B-empty mbarriers;
//   warps 4-7       : A producers (thread = channel = TMEM lane): value loads for the next
//                     chunk in flight while the current one is split and tcgen05.st'd
//                     into one of 4 TMEM stages;
//   warps 8-15      : B producers: weights of (in-reach block, cell, 4 samples) items into
//                     one of 2 SMEM stages (canonical K-major, no swizzle); per-chunk W
//                     partials reduced per cell in a fixed order (two-level, compensated);
//   dense mode      : every PROMOTE_CHUNKS chunks, at a bin-row boundary, warps 0-3 move D
//                     into the CTA's own (exclusively owned) out_map slice as fp32 partial
//                     sums and the MMAs restart D, so no TMEM accumulator ever sums more
//                     than ~10^3 MMA partials (tensor-core accumulation is not fp32-RN).
// Epilogue: tcgen05.ld of each block's D, V = S / W (IEEE div), NaN where W = 0.
// Deterministic: fixed chunk order, fixed work mapping, no atomics.
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "weight.cuh"

namespace hg {

constexpr int TC_THREADS = 512;
constexpr int TC_M = 128;                 // channels per CTA (UMMA M)
constexpr int TC_BX = 4, TC_BY = 4;       // blocks per CTA tile
constexpr int TC_NB = TC_BX * TC_BY;      // 16 blocks
constexpr int TC_N = 16;                  // cells per block (UMMA N): 4 x 4
constexpr int TC_TW = TC_BX * 4, TC_TH = TC_BY * 4;
constexpr int TC_KC = 32;                 // samples per chunk (4 MMA K-steps of 8)
constexpr int NA = 4;                     // A stages (TMEM)
constexpr int NBS = 2;                    // B stages (SMEM)
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t A_COL0 = TC_NB * TC_N; // 256: A stages after the accumulators
constexpr int B_TILE = TC_N * TC_KC * 4;  // 2 KB per hi or lo tile
constexpr int B_SLOT = 2 * B_TILE;
constexpr int B_STAGE = TC_NB * B_SLOT;   // 64 KB
constexpr uint32_t IDESC = tc::idesc_tf32(TC_M, TC_N);
constexpr int W_THREADS = 256;            // B producers (warps 8-15)
constexpr int PROMOTE_CHUNKS = 64;

struct TcSmem {
    uint8_t B[NBS][B_STAGE];
    float wpart[NBS][TC_NB][TC_N][TC_KC / 4];
    float Wfin[TC_NB * TC_N];
    uint64_t a_full[NA], a_empty[NA], b_full[NBS], b_empty[NBS];
    uint64_t bar_done, bar_prom;
    uint32_t tmem_base;
    uint32_t touched;
    int n_prom;
};

// byte offset of (cell n, sample k) inside one 16 x 32 tf32 B tile (k multiple of 4)
__device__ __forceinline__ uint32_t b_off(int n, int k) {
    return (uint32_t)((k >> 3) * 512 + ((k >> 2) & 1) * 256 + (n >> 3) * 128 + (n & 7) * 16);
}

// The chunk sequence of a CTA tile, identical in every role.
struct ChunkWalk {
    int br, br_end, m, rc;
    uint32_t p0, s1;
    int i0, j0, i_hi;
    __device__ void row_setup(const Geom& g, const PlanDev& pd) {
        m = pd.mrow[br];
        const int64_t rowb = (int64_t)br * g.ncol;
        p0 = pd.bin_start[rowb + i0 + g.mlon - m];
        s1 = pd.bin_start[rowb + i_hi + g.mlon + m + 1];
        rc = br - g.mlat;
    }
    __device__ void init(const Geom& g, const PlanDev& pd, int ti0, int tj0) {
        i0 = ti0;
        j0 = tj0;
        i_hi = min(i0 + TC_TW - 1, g.nx - 1);
        br = j0;
        br_end = min(j0 + TC_TH - 1, g.ny - 1) + 2 * g.mlat;
        row_setup(g, pd);
    }
    // Advance to the next chunk that reaches at least one block; returns false at the end.
    // new_row is set when the chunk is the first processed one of its bin row.
    __device__ bool next(const Geom& g, const PlanDev& pd, uint32_t& mask, uint32_t& pstart,
                         uint32_t& nk, int& row, bool& row_change) {
        row_change = false;
        while (true) {
            while (p0 >= s1) {
                if (++br > br_end) return false;
                row_setup(g, pd);
                row_change = true;
            }
            const uint32_t p = p0;
            const uint32_t n = min((uint32_t)TC_KC, s1 - p);
            p0 += TC_KC;
            const int bc_first = __float_as_int(pd.geo[p].w);
            const int bc_last = __float_as_int(pd.geo[p + n - 1].w);
            const int clo = bc_first - g.mlon - m, chi = bc_last - g.mlon + m;
            uint32_t mk = 0;
#pragma unroll
            for (int b = 0; b < TC_NB; ++b) {
                const int bi = i0 + (b % TC_BX) * 4, bj = j0 + (b / TC_BX) * 4;
                const bool rows = bj <= rc + g.rl && bj + 3 >= rc - g.rl && bj < g.ny;
                const bool cols = bi <= chi && bi + 3 >= clo && bi < g.nx;
                if (rows && cols) mk |= 1u << b;
            }
            if (mk) {
                mask = mk;
                pstart = p;
                nk = n;
                row = br;
                return true;
            }
        }
    }
};

template <bool PROMOTE>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_accum_tc(const __grid_constant__ Geom g, PlanDev pd, const float* __restrict__ V, int64_t ldv,
           int C, float* __restrict__ out, float* __restrict__ wout, int promote_every) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    TcSmem& sm = *reinterpret_cast<TcSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    const int i0 = (blockIdx.x % tiles_x) * TC_TW, j0 = (blockIdx.x / tiles_x) * TC_TH;
    const int cb = blockIdx.y * TC_M;

    if (warp == 0) tc::tmem_alloc(&sm.tmem_base, TMEM_COLS);
    if (tid == 32) {
        for (int s = 0; s < NA; ++s) {
            tc::mbar_init(&sm.a_full[s], 128);
            tc::mbar_init(&sm.a_empty[s], 1);
        }
        for (int s = 0; s < NBS; ++s) {
            tc::mbar_init(&sm.b_full[s], W_THREADS);
            tc::mbar_init(&sm.b_empty[s], 1);
        }
        tc::mbar_init(&sm.bar_done, 1);
        tc::mbar_init(&sm.bar_prom, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < W_THREADS) sm.Wfin[tid] = 0.0f;
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = sm.tmem_base;

    const int64_t cells = (int64_t)g.nx * g.ny;
    if constexpr (PROMOTE) {
        // the CTA's out slice holds the promoted fp32 partial sums: start from 0
        for (int e = tid; e < TC_M * TC_TW * TC_TH; e += TC_THREADS) {
            const int ch = cb + e / (TC_TW * TC_TH), cl = e % (TC_TW * TC_TH);
            const int i = i0 + cl % TC_TW, j = j0 + cl / TC_TW;
            if (ch < C && i < g.nx && j < g.ny) out[(int64_t)ch * cells + (int64_t)j * g.nx + i] = 0.0f;
        }
        __syncthreads();
    }
    // dense mode: D -> fp32 partial sums in this CTA's out slice (warps 0-3, lane quarter
    // = warp), all 16 blocks; first promotion writes, later ones add
    auto promote = [&](int nprom) {
        tc::mbar_wait(&sm.bar_prom, nprom & 1);
        tc::fence_after_sync();
        const uint32_t tm = sm.touched;
        const int ch = cb + warp * 32 + lane;
#pragma unroll 1
        for (int b = 0; b < TC_NB; ++b) {
            if (!((tm >> b) & 1)) continue;
            uint32_t r[16];
            tc::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(b * TC_N), r);
            tc::wait_ld();
            if (ch < C) {
                const int bi = i0 + (b % TC_BX) * 4, bj = j0 + (b / TC_BX) * 4;
#pragma unroll
                for (int n = 0; n < TC_N; ++n) {
                    const int i = bi + (n & 3), j = bj + (n >> 2);
                    if (i < g.nx && j < g.ny) {
                        float* o = out + (int64_t)ch * cells + (int64_t)j * g.nx + i;
                        *o += __uint_as_float(r[n]);
                    }
                }
            } else {
                (void)r;
            }
        }
        // blocks never touched since the start: their partial stays as is (or 0 below)
        tc::fence_before_sync();
    };

    ChunkWalk walk;
    walk.init(g, pd, i0, j0);
    uint32_t mask, pstart, nk;
    int row;
    bool row_change;
    int c = 0;                 // processed-chunk counter
    int since = 0;             // chunks since the last promotion (dense mode)
    int prom = 0;              // promotions so far

    if (warp == 0) {
        // ============================ MMA issuer =============================
        uint32_t touched = 0;
        while (walk.next(g, pd, mask, pstart, nk, row, row_change)) {
            if constexpr (PROMOTE) {
                if (since >= promote_every) {
                    // drain the tensor core, move D out (warps 0-3), restart D
                    if (lane == 0) {
                        sm.touched = touched;
                        tc::mma_commit(&sm.bar_prom);
                    }
                    __syncwarp();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    promote(prom);
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    touched = 0;
                    since = 0;
                    ++prom;
                }
            }
            const int sa = c % NA, sb = c % NBS;
            tc::mbar_wait(&sm.a_full[sa], (c / NA) & 1);
            tc::mbar_wait(&sm.b_full[sb], (c / NBS) & 1);
            tc::fence_after_sync();
            if (lane == 0) {
                const uint32_t bt0 = tc::smem_u32(&sm.B[sb][0]);
                uint32_t mm = mask;
                int q = 0;
                while (mm) {
                    const int b = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const uint32_t d = tmem + (uint32_t)(b * TC_N);
                    const uint32_t bt = bt0 + (uint32_t)(q * B_SLOT);
                    uint32_t acc = (touched >> b) & 1;
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 8; ++ks) {
                        const uint32_t ah = tmem + A_COL0 + sa * 64 + ks * 8;
                        const uint64_t bh = tc::sdesc(bt + ks * 512, 256, 128);
                        const uint64_t bl = tc::sdesc(bt + B_TILE + ks * 512, 256, 128);
                        tc::mma_tf32_ts(d, ah, bh, IDESC, acc);
                        tc::mma_tf32_ts(d, ah, bl, IDESC, 1);
                        tc::mma_tf32_ts(d, ah + 32, bh, IDESC, 1);
                        acc = 1;
                    }
                    touched |= 1u << b;
                    ++q;
                }
                tc::mma_commit(&sm.a_empty[sa]);
                tc::mma_commit(&sm.b_empty[sb]);
            }
            __syncwarp();
            ++c;
            ++since;
        }
        if (lane == 0) {
            sm.touched = touched;
            sm.n_prom = prom;
            tc::mma_commit(&sm.bar_done);
        }
        __syncwarp();
    } else if (warp >= 4 && warp < 8) {
        // ============================ A producers ============================
        const int q4 = warp & 3;
        const int ch = cb + q4 * 32 + lane;
        const bool ch_ok = ch < C;
        float vn[TC_KC];
        bool have = walk.next(g, pd, mask, pstart, nk, row, row_change);
        if (have) {
#pragma unroll
            for (int k = 0; k < TC_KC; ++k)
                vn[k] = ((uint32_t)k < nk && ch_ok) ? __ldg(V + (int64_t)(pstart + k) * ldv + ch) : 0.0f;
        }
        while (have) {
            uint32_t hi[TC_KC], lo[TC_KC];
#pragma unroll
            for (int k = 0; k < TC_KC; ++k) {
                hi[k] = tc::to_tf32(vn[k]);
                lo[k] = tc::to_tf32(vn[k] - __uint_as_float(hi[k]));
            }
            // prefetch the next chunk's values while this one is stored
            have = walk.next(g, pd, mask, pstart, nk, row, row_change);
            if (have) {
#pragma unroll
                for (int k = 0; k < TC_KC; ++k)
                    vn[k] = ((uint32_t)k < nk && ch_ok) ? __ldg(V + (int64_t)(pstart + k) * ldv + ch)
                                                       : 0.0f;
            }
            const int sa = c % NA;
            if (c >= NA) tc::mbar_wait(&sm.a_empty[sa], ((c / NA) - 1) & 1);
            tc::fence_after_sync();
            const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + A_COL0 + sa * 64;
            tc::tmem_st32(ta, hi);
            tc::tmem_st32(ta + 32, lo);
            tc::wait_st();
            tc::fence_before_sync();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                         :: "r"(tc::smem_u32(&sm.a_full[sa])) : "memory");
            ++c;
        }
    } else if (warp >= 8) {
        // ============================ B producers ============================
        const int wt = tid - 8 * 32;                  // 0..255
        // W ownership: thread wt owns cell (wb, wn) of the tile
        const int wb = wt >> 4, wn = wt & 15;
        const int ci_own = i0 + (wb % TC_BX) * 4 + (wn & 3);
        const int cj_own = j0 + (wb / TC_BX) * 4 + (wn >> 2);
        float Wsum = 0.0f, Wc = 0.0f;
        while (walk.next(g, pd, mask, pstart, nk, row, row_change)) {
            const int sb = c % NBS;
            if (c >= NBS) tc::mbar_wait(&sm.b_empty[sb], ((c / NBS) - 1) & 1);
            const int nq = __popc(mask);
            // items: (slot q, cell n, sample quad) ; 128 per slot
            for (int it = wt; it < nq * 128; it += W_THREADS) {
                const int q = it >> 7, n = (it >> 3) & 15, kq = it & 7;
                // q-th set bit of mask -> block b
                uint32_t mm = mask;
                for (int z = 0; z < q; ++z) mm &= mm - 1;
                const int b = __ffs(mm) - 1;
                const int ci = i0 + (b % TC_BX) * 4 + (n & 3);
                const int cj = j0 + (b / TC_BX) * 4 + (n >> 2);
                const bool ok = ci < g.nx && cj < g.ny;
                const float cos_c = ok ? pd.cos_row[cj] : 1.0f;
                float w4[4];
                float part = 0.0f;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = kq * 4 + u;
                    float w = 0.0f;
                    if (ok && (uint32_t)k < nk)
                        w = pair_weight(g, pd, ci, cj, cos_c, row, pd.geo[pstart + k],
                                        (int)(pstart + k));
                    w4[u] = w;
                    part += w;
                }
                uint4 h, l;
                h.x = tc::to_tf32(w4[0]); l.x = tc::to_tf32(w4[0] - __uint_as_float(h.x));
                h.y = tc::to_tf32(w4[1]); l.y = tc::to_tf32(w4[1] - __uint_as_float(h.y));
                h.z = tc::to_tf32(w4[2]); l.z = tc::to_tf32(w4[2] - __uint_as_float(h.z));
                h.w = tc::to_tf32(w4[3]); l.w = tc::to_tf32(w4[3] - __uint_as_float(h.w));
                uint8_t* tile = &sm.B[sb][q * B_SLOT];
                *reinterpret_cast<uint4*>(tile + b_off(n, kq * 4)) = h;
                *reinterpret_cast<uint4*>(tile + B_TILE + b_off(n, kq * 4)) = l;
                sm.wpart[sb][q][n][kq] = part;
            }
            asm volatile("bar.sync 2, 256;" ::: "memory");          // B producers only
            if ((mask >> wb) & 1) {
                const int q = __popc(mask & ((1u << wb) - 1));
                float s = 0.0f;
#pragma unroll
                for (int kq = 0; kq < TC_KC / 4; ++kq) s += sm.wpart[sb][q][wn][kq];
                const float y = s - Wc;                          // compensated outer sum
                const float t = Wsum + y;
                Wc = (t - Wsum) - y;
                Wsum = t;
            }
            tc::fence_proxy_async_smem();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                         :: "r"(tc::smem_u32(&sm.b_full[sb])) : "memory");
            ++c;
        }
        (void)ci_own;
        (void)cj_own;
        sm.Wfin[wt] = Wsum;
    }

    // ---- dense mode: warps 1-3 follow the issuer's promotion decisions
    if constexpr (PROMOTE) {
        if (warp >= 1 && warp < 4) {
            int since2 = 0;
            while (walk.next(g, pd, mask, pstart, nk, row, row_change)) {
                if (since2 >= promote_every) {
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    promote(prom);
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    since2 = 0;
                    ++prom;
                }
                ++since2;
            }
        }
    }

    __syncthreads();
    // ---- epilogue: wait for the last MMAs
    tc::mbar_wait(&sm.bar_done, 0);
    tc::fence_after_sync();
    const uint32_t tmask = sm.touched;
    const int prom_total = sm.n_prom;
    (void)prom_total;
    const float qnan = __int_as_float(0x7fc00000);
    if (warp < 8) {
        const int ch = cb + (warp & 3) * 32 + lane;
        const int half = warp >> 2;
#pragma unroll 1
        for (int a = 0; a < 8; ++a) {
            const int b = half * 8 + a;
            uint32_t r[16];
            const bool tb = (tmask >> b) & 1;
            if (tb) {
                tc::tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(b * TC_N), r);
                tc::wait_ld();
            }
            if (ch < C) {
                const int bi = i0 + (b % TC_BX) * 4, bj = j0 + (b / TC_BX) * 4;
#pragma unroll
                for (int n = 0; n < TC_N; ++n) {
                    const int i = bi + (n & 3), j = bj + (n >> 2);
                    if (i < g.nx && j < g.ny) {
                        float* o = out + (int64_t)ch * cells + (int64_t)j * g.nx + i;
                        float S = tb ? __uint_as_float(r[n]) : 0.0f;
                        if constexpr (PROMOTE) S += *o;
                        const float W = sm.Wfin[b * TC_N + n];
                        *o = W > 0.0f ? __fdiv_rn(S, W) : qnan;
                    }
                }
            }
        }
    }
    if (blockIdx.y == 0 && wout != nullptr && tid < W_THREADS) {
        const int b = tid >> 4, n = tid & 15;
        const int i = i0 + (b % TC_BX) * 4 + (n & 3), j = j0 + (b / TC_BX) * 4 + (n >> 2);
        if (i < g.nx && j < g.ny) wout[(int64_t)j * g.nx + i] = sm.Wfin[tid];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, TMEM_COLS);
}

hegrid_status launch_accumulate_tc(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                   int64_t n_channels, float* d_out, float* d_weight,
                                   cudaStream_t st) {
    if (n_channels <= 0) return HEGRID_OK;
    if (n_channels > (1LL << 30)) return HEGRID_EINVAL;
    const Geom& g = p->g;
    int C = (int)n_channels;
    int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    dim3 grid(tiles, (C + TC_M - 1) / TC_M);
    size_t smem = sizeof(TcSmem);
    const bool dense = p->max_cand > 4096;
    int promote_every = 32;
    if (const char* e = getenv("HEGRID_TC_PROMOTE")) promote_every = atoi(e) > 0 ? atoi(e) : 1 << 30;
    if (dense) {
        HG_TRY(cudaFuncSetAttribute(k_accum_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
        k_accum_tc<true><<<grid, TC_THREADS, smem, st>>>(g, p->dev(), d_v, ldv, C, d_out, d_weight,
                                                            promote_every);
    } else {
        HG_TRY(cudaFuncSetAttribute(k_accum_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
        k_accum_tc<false><<<grid, TC_THREADS, smem, st>>>(g, p->dev(), d_v, ldv, C, d_out, d_weight,
                                                            promote_every);
    }
    count_launch();
    return cuda_status(cudaGetLastError());
}

}  // namespace hg
