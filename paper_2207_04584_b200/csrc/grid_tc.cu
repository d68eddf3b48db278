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
// CTA = 16x16 cells (16 blocks) x 128 channels, 256 threads:
//   warps 0-3 : stage A (thread = channel lane): load 32 samples x its channel, split,
//               tcgen05.st into the stage's TMEM columns;
//   all warps : weights of in-reach blocks (thread = one cell of one block) -> SMEM in the
//               canonical K-major no-swizzle UMMA layout; W partials (two-level sum);
//   thread 0  : issues the MMAs of the chunk (only blocks the chunk can reach) and commits
//               them to the stage's mbarrier; two stages double-buffer A (TMEM) and B (SMEM)
//               so the tensor core runs chunk c while the SIMT warps prepare chunk c+1.
// Epilogue: tcgen05.ld of each block's D, V = S / W (IEEE div), NaN where W = 0.
// Deterministic: fixed chunk order and fixed thread->cell mapping; no atomics.
#include "common.cuh"
#include "tc_ptx.cuh"
#include "weight.cuh"

namespace hg {

constexpr int TC_THREADS = 256;
constexpr int TC_M = 128;                 // channels per CTA (UMMA M)
constexpr int TC_BX = 4, TC_BY = 4;       // blocks per CTA tile
constexpr int TC_NB = TC_BX * TC_BY;      // 16 blocks
constexpr int TC_N = 16;                  // cells per block (UMMA N): 4 x 4
constexpr int TC_TW = TC_BX * 4, TC_TH = TC_BY * 4;
constexpr int TC_KC = 32;                 // samples per chunk (4 MMA K-steps of 8)
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t A_COL0 = TC_NB * TC_N;  // 256: A stages after the accumulators
constexpr int B_TILE = TC_N * TC_KC * 4;  // 2 KB per hi or lo tile
constexpr int B_SLOT = 2 * B_TILE;
constexpr int B_STAGE = TC_NB * B_SLOT;   // 64 KB
constexpr uint32_t IDESC = tc::idesc_tf32(TC_M, TC_N);

struct TcSmem {
    uint8_t B[2][B_STAGE];
    float Wfin[TC_NB * TC_N];
    uint64_t bar[2];
    uint64_t bar_done;
    uint32_t tmem_base;
    uint32_t touched;
};

// byte offset of (cell n, sample k) inside one 16 x 32 tf32 B tile (k multiple of 4)
__device__ __forceinline__ uint32_t b_off(int n, int k) {
    return (uint32_t)((k >> 3) * 512 + ((k >> 2) & 1) * 256 + (n >> 3) * 128 + (n & 7) * 16);
}

__global__ void __launch_bounds__(TC_THREADS, 1)
k_accum_tc(const __grid_constant__ Geom g, PlanDev pd, const float* __restrict__ V, int64_t ldv,
           int C, float* __restrict__ out, float* __restrict__ wout) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    TcSmem& sm = *reinterpret_cast<TcSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    const int i0 = (blockIdx.x % tiles_x) * TC_TW, j0 = (blockIdx.x / tiles_x) * TC_TH;
    const int cb = blockIdx.y * TC_M;

    if (warp == 0) tc::tmem_alloc(&sm.tmem_base, TMEM_COLS);
    if (tid == 0) {
        tc::mbar_init(&sm.bar[0], 1);
        tc::mbar_init(&sm.bar[1], 1);
        tc::mbar_init(&sm.bar_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t b_base = tc::smem_u32(&sm.B[0][0]);

    // this thread's cell for weights / W: block wb, cell wn
    const int wb = tid >> 4, wn = tid & 15;
    const int ci = i0 + (wb % TC_BX) * 4 + (wn & 3);
    const int cj = j0 + (wb / TC_BX) * 4 + (wn >> 2);
    const bool cell_ok = ci < g.nx && cj < g.ny;
    const float cos_c = cell_ok ? pd.cos_row[cj] : 1.0f;
    float Wsum = 0.0f, Wc = 0.0f;            // Kahan-compensated outer sum
    uint32_t touched = 0;                    // thread 0: blocks with accumulated D

    const int i_hi = min(i0 + TC_TW - 1, g.nx - 1), j_hi = min(j0 + TC_TH - 1, g.ny - 1);
    int chunk = 0;
    for (int br = j0; br <= j_hi + 2 * g.mlat; ++br) {
        const int m = pd.mrow[br];
        const int64_t rowb = (int64_t)br * g.ncol;
        const uint32_t s0 = pd.bin_start[rowb + i0 + g.mlon - m];
        const uint32_t s1 = pd.bin_start[rowb + i_hi + g.mlon + m + 1];
        const int rc = br - g.mlat;          // cell row of this bin row
        for (uint32_t p0 = s0; p0 < s1; p0 += TC_KC) {
            const int st = chunk & 1;
            const uint32_t nk = min((uint32_t)TC_KC, s1 - p0);
            // blocks this chunk can reach (uniform across the CTA)
            const int bc_first = __float_as_int(pd.geo[p0].w);
            const int bc_last = __float_as_int(pd.geo[p0 + nk - 1].w);
            const int clo = bc_first - g.mlon - m, chi = bc_last - g.mlon + m;
            uint32_t mask = 0;
#pragma unroll
            for (int b = 0; b < TC_NB; ++b) {
                const int bi = i0 + (b % TC_BX) * 4, bj = j0 + (b / TC_BX) * 4;
                const bool rows = bj <= rc + g.rl && bj + 3 >= rc - g.rl && bj < g.ny;
                const bool cols = bi <= chi && bi + 3 >= clo && bi < g.nx;
                if (rows && cols) mask |= 1u << b;
            }
            if (mask == 0) continue;
            // stage free? (MMAs of chunk - 2 done)
            if (chunk >= 2) {
                tc::mbar_wait(&sm.bar[st], ((chunk - 2) >> 1) & 1);
                tc::fence_after_sync();
            }
            // ---- A: values, thread = channel lane (warps 0-3)
            if (warp < 4) {
                const int ch = cb + warp * 32 + lane;
                uint32_t hi[32], lo[32];
#pragma unroll
                for (int k = 0; k < TC_KC; ++k) {
                    float v = 0.0f;
                    if ((uint32_t)k < nk && ch < C) v = __ldg(V + (int64_t)(p0 + k) * ldv + ch);
                    hi[k] = tc::to_tf32(v);
                    lo[k] = tc::to_tf32(v - __uint_as_float(hi[k]));
                }
                const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + A_COL0 + st * 64;
                tc::tmem_st32(ta, hi);
                tc::tmem_st32(ta + 32, lo);
                tc::wait_st();
            }
            // ---- B: weights of this thread's cell for the chunk's samples
            if ((mask >> wb) & 1) {
                const int q = __popc(mask & ((1u << wb) - 1));
                uint8_t* tile = &sm.B[st][q * B_SLOT];
                float wpart = 0.0f;
#pragma unroll 2
                for (int k = 0; k < TC_KC; k += 4) {
                    float w4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t p = p0 + k + u;
                        float w = 0.0f;
                        if (cell_ok && (uint32_t)(k + u) < nk)
                            w = pair_weight(g, pd, ci, cj, cos_c, br, pd.geo[p], (int)p);
                        w4[u] = w;
                        wpart += w;
                    }
                    uint4 h, l;
                    h.x = tc::to_tf32(w4[0]); l.x = tc::to_tf32(w4[0] - __uint_as_float(h.x));
                    h.y = tc::to_tf32(w4[1]); l.y = tc::to_tf32(w4[1] - __uint_as_float(h.y));
                    h.z = tc::to_tf32(w4[2]); l.z = tc::to_tf32(w4[2] - __uint_as_float(h.z));
                    h.w = tc::to_tf32(w4[3]); l.w = tc::to_tf32(w4[3] - __uint_as_float(h.w));
                    *reinterpret_cast<uint4*>(tile + b_off(wn, k)) = h;
                    *reinterpret_cast<uint4*>(tile + B_TILE + b_off(wn, k)) = l;
                }
                // two-level W: chunk partial into a compensated running sum
                const float y = wpart - Wc;
                const float t = Wsum + y;
                Wc = (t - Wsum) - y;
                Wsum = t;
            }
            tc::fence_proxy_async_smem();
            tc::fence_before_sync();
            __syncthreads();
            if (tid == 0) {
                tc::fence_after_sync();
                uint32_t mm = mask;
                int q = 0;
                while (mm) {
                    const int b = __ffs(mm) - 1;
                    mm &= mm - 1;
                    const uint32_t d = tmem + (uint32_t)(b * TC_N);
                    const uint32_t bt = b_base + (uint32_t)(st * B_STAGE + q * B_SLOT);
                    uint32_t acc = (touched >> b) & 1;
#pragma unroll
                    for (int ks = 0; ks < TC_KC / 8; ++ks) {
                        const uint32_t ah = tmem + A_COL0 + st * 64 + ks * 8;
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
                tc::mma_commit(&sm.bar[st]);
            }
            ++chunk;
        }
    }
    // ---- drain: all MMAs complete
    if (tid == 0) {
        tc::mma_commit(&sm.bar_done);
        sm.touched = touched;
    }
    sm.Wfin[tid] = Wsum;
    __syncthreads();
    tc::mbar_wait(&sm.bar_done, 0);
    tc::fence_after_sync();
    const uint32_t tmask = sm.touched;

    // ---- epilogue: warp w reads TMEM lanes 32*(w%4).. (its channels), blocks of half w/4
    const float qnan = __int_as_float(0x7fc00000);
    const int64_t cells = (int64_t)g.nx * g.ny;
    const int ch = cb + (warp & 3) * 32 + lane;
    for (int b = (warp >> 2) * (TC_NB / 2); b < ((warp >> 2) + 1) * (TC_NB / 2); ++b) {
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
                    const float W = sm.Wfin[b * TC_N + n];
                    const float S = tb ? __uint_as_float(r[n]) : 0.0f;
                    out[(int64_t)ch * cells + (int64_t)j * g.nx + i] = W > 0.0f ? __fdiv_rn(S, W) : qnan;
                }
            }
        }
    }
    if (blockIdx.y == 0 && wout != nullptr && cell_ok) wout[(int64_t)cj * g.nx + ci] = Wsum;
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
    size_t smem = sizeof(TcSmem) + 1024;
    HG_TRY(cudaFuncSetAttribute(k_accum_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_accum_tc<<<grid, TC_THREADS, smem, st>>>(g, p->dev(), d_v, ldv, C, d_out, d_weight);
    count_launch();
    return cuda_status(cudaGetLastError());
}

}  // namespace hg
