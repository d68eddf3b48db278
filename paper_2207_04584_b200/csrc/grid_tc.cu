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
// The per-tile chunk sequence (bin rows of the tile's reach, 32-sample chunks, and which
// of the tile's 16 blocks each chunk can reach) is part of the plan: built once on the
// device by k_tc_schedule and read by every role of every launch (Algorithm 1's
// "determine the region ... of the contribution points", hoisted out of
// the hot loop and shared by all channels).
//
// CTA = 16x16 cells (16 blocks) x 128 channels, 512 threads, warp-specialised:
//   warp 0 (lane 0) : MMA issuer.  Waits A-full and B-full of a stage, issues 12 MMAs per
//                     in-reach block, commits to the A-empty and B-empty mbarriers;
//   warps 4-7       : A producers (thread = channel = TMEM lane): the next chunk's values
//                     are in flight while the current one is split and tcgen05.st'd into
//                     one of 4 TMEM stages;
//   warps 8-15      : B producers: thread = (cell row, 4-sample quad, slots q0, q0+8); the
//                     quad's sample geometry is prefetched a chunk ahead; weights go to one
//                     of 3 SMEM stages (canonical K-major, no swizzle); per-cell W partials
//                     are reduced in a fixed order (two-level, compensated);
//   dense mode      : every `promote_every` chunks warps 0-3 move D into the CTA's own
//                     (exclusively owned) out_map slice as fp32 partial sums and the MMAs
//                     restart D, bounding the number of tensor-core accumulations (which
//                     are not fp32 round-to-nearest) behind any partial sum.
// Epilogue: tcgen05.ld of each block's D, V = S / W (IEEE div), NaN where W = 0.
// Deterministic: fixed chunk order, fixed work mapping, no atomics.
#include <stdlib.h>

#include <vector>

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
constexpr int NBS = 3;                    // B stages (SMEM)
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t A_COL0 = TC_NB * TC_N; // 256: A stages after the accumulators
constexpr int B_TILE = TC_N * TC_KC * 4;  // 2 KB per hi or lo tile
constexpr int B_SLOT = 2 * B_TILE;
constexpr int B_STAGE = TC_NB * B_SLOT;   // 64 KB
constexpr uint32_t IDESC = tc::idesc_tf32(TC_M, TC_N);
constexpr int W_THREADS = 256;            // B producers (warps 8-15)

struct TcSmem {
    uint8_t B[NBS][B_STAGE];
    float wpart[NBS][TC_NB][TC_N][TC_KC / 4];
    float Wfin[TC_NB * TC_N];
    uint64_t a_full[NA], a_empty[NA], b_full[NBS], b_empty[NBS];
    uint64_t bar_done, bar_prom;
    uint32_t tmem_base;
    uint32_t touched;
};

// byte offset of (cell n, sample k) inside one 16 x 32 tf32 B tile (k multiple of 4)
__device__ __forceinline__ uint32_t b_off(int n, int k) {
    return (uint32_t)((k >> 3) * 512 + ((k >> 2) & 1) * 256 + (n >> 3) * 128 + (n & 7) * 16);
}

// ------------------------------------------------------------------ chunk schedule
// One warp per tile; lanes evaluate 32 consecutive chunks of a bin row at once.
// n_out != nullptr: count only; otherwise write entries at off[tile].
__global__ void k_tc_schedule(const __grid_constant__ Geom g, PlanDev pd, int tiles,
                              uint32_t* __restrict__ n_out, const uint32_t* __restrict__ off,
                              uint4* __restrict__ sched) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= tiles) return;
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    const int i0 = (warp % tiles_x) * TC_TW, j0 = (warp / tiles_x) * TC_TH;
    const int i_hi = min(i0 + TC_TW - 1, g.nx - 1);
    const int br_end = min(j0 + TC_TH - 1, g.ny - 1) + 2 * g.mlat;
    uint32_t cnt = 0;
    const uint32_t base = n_out ? 0 : off[warp];
    for (int br = j0; br <= br_end; ++br) {
        const int m = pd.mrow[br];
        const int64_t rowb = (int64_t)br * g.ncol;
        const uint32_t s0 = pd.bin_start[rowb + i0 + g.mlon - m];
        const uint32_t s1 = pd.bin_start[rowb + i_hi + g.mlon + m + 1];
        const int rc = br - g.mlat;
        for (uint32_t c0 = s0; c0 < s1; c0 += 32u * TC_KC) {
            const uint32_t p = c0 + (uint32_t)lane * TC_KC;
            uint32_t mk = 0, n = 0;
            if (p < s1) {
                n = min((uint32_t)TC_KC, s1 - p);
                const int clo = __float_as_int(pd.geo[p].w) - g.mlon - m;
                const int chi = __float_as_int(pd.geo[p + n - 1].w) - g.mlon + m;
#pragma unroll
                for (int b = 0; b < TC_NB; ++b) {
                    const int bi = i0 + (b % TC_BX) * 4, bj = j0 + (b / TC_BX) * 4;
                    const bool rows = bj <= rc + g.rl && bj + 3 >= rc - g.rl && bj < g.ny;
                    const bool cols = bi <= chi && bi + 3 >= clo && bi < g.nx;
                    if (rows && cols) mk |= 1u << b;
                }
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, mk != 0);
            if (mk && sched) {
                const uint32_t pos = base + cnt + __popc(bal & ((1u << lane) - 1));
                sched[pos] = make_uint4(p, n, (uint32_t)br, mk);
            }
            cnt += __popc(bal);
        }
    }
    if (n_out && lane == 0) n_out[warp] = cnt;
}

static hegrid_status ensure_tc_schedule(const hegrid_plan_s* p, cudaStream_t st) {
    if (p->tc_nchunks >= 0) return HEGRID_OK;
    const Geom& g = p->g;
    const int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    uint32_t* d_n = nullptr;
    HG_TRY(cudaMalloc(&d_n, (tiles + 1) * sizeof(uint32_t)));
    const int threads = 128, blocks = (tiles * 32 + threads - 1) / threads;
    k_tc_schedule<<<blocks, threads, 0, st>>>(g, p->dev(), tiles, d_n, nullptr, nullptr);
    count_launch();
    std::vector<uint32_t> h(tiles + 1, 0);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d_n, tiles * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFree(d_n);
        return cuda_status(e);
    }
    std::vector<uint32_t> off(tiles + 1, 0);
    for (int t = 0; t < tiles; ++t) off[t + 1] = off[t] + h[t];
    const int64_t total = off[tiles];
    uint4* d_s = nullptr;
    e = cudaMalloc(&d_s, std::max<int64_t>(total, 1) * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_n, off.data(), (tiles + 1) * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        k_tc_schedule<<<blocks, threads, 0, st>>>(g, p->dev(), tiles, nullptr, d_n, d_s);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFree(d_n);
        if (d_s) cudaFree(d_s);
        return cuda_status(e);
    }
    p->d_tc_sched = d_s;
    p->d_tc_tile_off = d_n;
    p->tc_nchunks = total;
    return HEGRID_OK;
}

// ------------------------------------------------------------------ the kernel
template <bool PROMOTE>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_accum_tc(const __grid_constant__ Geom g, PlanDev pd, const uint4* __restrict__ sched,
           const uint32_t* __restrict__ tile_off, const float* __restrict__ V, int64_t ldv,
           int C, float* __restrict__ out, float* __restrict__ wout, int promote_every, int dbg) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    TcSmem& sm = *reinterpret_cast<TcSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    const int i0 = (blockIdx.x % tiles_x) * TC_TW, j0 = (blockIdx.x / tiles_x) * TC_TH;
    const int cb = blockIdx.y * TC_M;
    const uint4* cs = sched + tile_off[blockIdx.x];
    const int nchunks = (int)(tile_off[blockIdx.x + 1] - tile_off[blockIdx.x]);
    const int64_t cells = (int64_t)g.nx * g.ny;

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
    if constexpr (PROMOTE) {
        // the CTA's out slice accumulates the promoted fp32 partial sums: start from 0
        for (int e = tid; e < TC_M * TC_TW * TC_TH; e += TC_THREADS) {
            const int ch = cb + e / (TC_TW * TC_TH), cl = e % (TC_TW * TC_TH);
            const int i = i0 + cl % TC_TW, j = j0 + cl / TC_TW;
            if (ch < C && i < g.nx && j < g.ny) out[(int64_t)ch * cells + (int64_t)j * g.nx + i] = 0.0f;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = sm.tmem_base;

    // dense mode: D -> this CTA's out slice (warps 0-3; lane quarter = warp)
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
                    if (i < g.nx && j < g.ny) out[(int64_t)ch * cells + (int64_t)j * g.nx + i] += __uint_as_float(r[n]);
                }
            }
        }
        tc::fence_before_sync();
    };

    if (warp == 0) {
        // ============================ MMA issuer =============================
        uint32_t touched = 0;
        int since = 0, prom = 0;
        for (int c = 0; c < nchunks; ++c) {
            const uint32_t mask = __ldg(&cs[c].w);
            if constexpr (PROMOTE) {
                if (since >= promote_every) {
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
            if (lane == 0 && !(dbg & 2)) {
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
            }
            if (lane == 0) {
                tc::mma_commit(&sm.a_empty[sa]);
                tc::mma_commit(&sm.b_empty[sb]);
            }
            __syncwarp();
            ++since;
        }
        if (lane == 0) {
            sm.touched = touched;
            tc::mma_commit(&sm.bar_done);
        }
        __syncwarp();
    } else if (warp < 4) {
        // ============================ dense mode: promotion helpers ==========
        if constexpr (PROMOTE) {
            int since = 0, prom = 0;
            for (int c = 0; c < nchunks; ++c) {
                if (since >= promote_every) {
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    promote(prom);
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    since = 0;
                    ++prom;
                }
                ++since;
            }
        }
    } else if (warp < 8) {
        // ============================ A producers ============================
        const int q4 = warp & 3;
        const int ch = cb + q4 * 32 + lane;
        const bool ch_ok = ch < C;
        float vn[TC_KC];
        const bool ch_ld = ch_ok && !(dbg & 4);
        if (nchunks > 0) {
            const uint4 e = __ldg(&cs[0]);
#pragma unroll
            for (int k = 0; k < TC_KC; ++k)
                vn[k] = ((uint32_t)k < e.y && ch_ld) ? __ldg(V + (int64_t)(e.x + k) * ldv + ch) : 0.0f;
        }
        for (int c = 0; c < nchunks; ++c) {
            uint32_t hi[TC_KC], lo[TC_KC];
#pragma unroll
            for (int k = 0; k < TC_KC; ++k) {
                hi[k] = tc::to_tf32(vn[k]);
                lo[k] = tc::to_tf32(vn[k] - __uint_as_float(hi[k]));
            }
            if (c + 1 < nchunks) {          // next chunk's values in flight
                const uint4 e = __ldg(&cs[c + 1]);
#pragma unroll
                for (int k = 0; k < TC_KC; ++k)
                    vn[k] = ((uint32_t)k < e.y && ch_ld) ? __ldg(V + (int64_t)(e.x + k) * ldv + ch) : 0.0f;
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
        }
    } else {
        // ============================ B producers ============================
        const int wt = tid - 8 * 32;                  // 0..255
        const int kq = wt & 7, rr = (wt >> 3) & 3, q0 = wt >> 5;
        // W ownership: thread wt owns cell (wb, wn) of the tile
        const int wb = wt >> 4, wn = wt & 15;
        float Wsum = 0.0f, Wc = 0.0f;
        const float hlon = 0.5f * g.dlon_rad, hlat = 0.5f * g.dlat_rad;
        float4 gq[4];
        uint4 e = make_uint4(0, 0, 0, 0);
        if (nchunks > 0) {
            e = __ldg(&cs[0]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                gq[u] = (uint32_t)(4 * kq + u) < e.y ? __ldg(&pd.geo[e.x + 4 * kq + u]) : make_float4(0, 0, 0, 0);
        }
        for (int c = 0; c < nchunks; ++c) {
            const uint32_t pstart = e.x, nk = e.y, mask = e.w;
            const int row = (int)e.z;
            float4 g4[4] = {gq[0], gq[1], gq[2], gq[3]};
            if (c + 1 < nchunks) {           // next chunk's geometry in flight
                e = __ldg(&cs[c + 1]);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    gq[u] = (uint32_t)(4 * kq + u) < e.y ? __ldg(&pd.geo[e.x + 4 * kq + u]) : make_float4(0, 0, 0, 0);
            }
            const int sb = c % NBS;
            if (c >= NBS) tc::mbar_wait(&sm.b_empty[sb], ((c / NBS) - 1) & 1);
            const int nq = (dbg & 1) ? 0 : __popc(mask);
#pragma unroll 1
            for (int q = q0; q < nq; q += 8) {
                const int b = __fns(mask, 0, q + 1);
                const int cj = j0 + (b / TC_BX) * 4 + rr;
                const int ci0 = i0 + (b % TC_BX) * 4;
                const bool rok = cj < g.ny;
                const float cos_c = rok ? pd.cos_row[cj] : 1.0f;
                float w[4][4];                 // [cell col][sample]
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 s = g4[u];
                    const bool sok = rok && (uint32_t)(4 * kq + u) < nk;
                    const float dy = (float)(row - g.mlat - cj) + s.y;
                    const float a = dy * hlat;
                    const float a2 = a * a;
                    const float sa = fmaf(a2 * (-1.0f / 3.0f), a2, a2);
                    const float ccs = cos_c * s.z;
                    const float dx0 = (float)(__float_as_int(s.w) - g.mlon - ci0) + s.x;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const float bb = (dx0 - (float)cc) * hlon;
                        const float b2 = bb * bb;
                        const float sbv = fmaf(b2 * (-1.0f / 3.0f), b2, b2);
                        const float h = fmaf(ccs, sbv, sa);
                        const float d2 = (4.0f * h) * fmaf(h, fmaf(h, 8.0f / 45.0f, 1.0f / 3.0f), 1.0f);
                        const bool cok = sok && (ci0 + cc < g.nx);
                        bool in = d2 <= g.R2_lo;
                        if (!in && d2 <= g.R2_hi && cok) {
                            const double2 ll = pd.ll[pstart + 4 * kq + u];
                            in = support_fp64(g, ci0 + cc, cj, ll.x, ll.y);
                        }
                        w[cc][u] = (in && cok) ? ex2_approx(d2 * g.neg_k2) : 0.0f;
                    }
                }
                uint8_t* tile = &sm.B[sb][q * B_SLOT];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int n = rr * 4 + cc;
                    uint4 h4, l4;
                    h4.x = tc::to_tf32(w[cc][0]); l4.x = tc::to_tf32(w[cc][0] - __uint_as_float(h4.x));
                    h4.y = tc::to_tf32(w[cc][1]); l4.y = tc::to_tf32(w[cc][1] - __uint_as_float(h4.y));
                    h4.z = tc::to_tf32(w[cc][2]); l4.z = tc::to_tf32(w[cc][2] - __uint_as_float(h4.z));
                    h4.w = tc::to_tf32(w[cc][3]); l4.w = tc::to_tf32(w[cc][3] - __uint_as_float(h4.w));
                    *reinterpret_cast<uint4*>(tile + b_off(n, kq * 4)) = h4;
                    *reinterpret_cast<uint4*>(tile + B_TILE + b_off(n, kq * 4)) = l4;
                    sm.wpart[sb][q][n][kq] = (w[cc][0] + w[cc][1]) + (w[cc][2] + w[cc][3]);
                }
            }
            tc::fence_proxy_async_smem();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                         :: "r"(tc::smem_u32(&sm.b_full[sb])) : "memory");
            asm volatile("bar.sync 2, 256;" ::: "memory");          // wpart complete
            if ((mask >> wb) & 1) {
                const int q = __popc(mask & ((1u << wb) - 1));
                float s = 0.0f;
#pragma unroll
                for (int k = 0; k < TC_KC / 4; ++k) s += sm.wpart[sb][q][wn][k];
                const float y = s - Wc;                          // compensated outer sum
                const float t = Wsum + y;
                Wc = (t - Wsum) - y;
                Wsum = t;
            }
        }
        sm.Wfin[wt] = Wsum;
    }

    __syncthreads();
    // ---- epilogue: wait for the last MMAs
    tc::mbar_wait(&sm.bar_done, 0);
    tc::fence_after_sync();
    const uint32_t tmask = sm.touched;
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
    HG_TRY_S(ensure_tc_schedule(p, st));
    const Geom& g = p->g;
    int C = (int)n_channels;
    int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    dim3 grid(tiles, (C + TC_M - 1) / TC_M);
    size_t smem = sizeof(TcSmem);
    const bool dense = p->max_cand > 4096;
    int promote_every = 16;
    int dbg = 0;
    if (const char* e = getenv("HEGRID_TC_DEBUG")) dbg = atoi(e);
    if (const char* e = getenv("HEGRID_TC_PROMOTE")) promote_every = atoi(e) > 0 ? atoi(e) : 1 << 30;
    if (dense) {
        HG_TRY(cudaFuncSetAttribute(k_accum_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
        k_accum_tc<true><<<grid, TC_THREADS, smem, st>>>(g, p->dev(), p->d_tc_sched,
                                                          p->d_tc_tile_off, d_v, ldv, C, d_out,
                                                          d_weight, promote_every, dbg);
    } else {
        HG_TRY(cudaFuncSetAttribute(k_accum_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
        k_accum_tc<false><<<grid, TC_THREADS, smem, st>>>(g, p->dev(), p->d_tc_sched,
                                                           p->d_tc_tile_off, d_v, ldv, C, d_out,
                                                           d_weight, promote_every, dbg);
    }
    count_launch();
    return cuda_status(cudaGetLastError());
}

}  // namespace hg
