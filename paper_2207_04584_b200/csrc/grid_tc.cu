// grid_tc.cu -- accumulate + normalise on the 5th-gen tensor cores (tcgen05: kind::tf32 and
// kind::f16), error-compensated so the sums keep fp32 accuracy.
//
// The contraction (Eq. 1 numerator): S[c][cell] = sum_n v[c][n] w(cell,n).
// Blocked: for a chunk of K = 32 plan-ordered candidate samples of one bin row and a run
// of r consecutive in-reach 4x4-cell blocks,
//     D[128 ch][16 r cells] += A[128 ch][32 samples] * B[16 r cells][32 samples]^T
// with A = the chunk's values (channels on TMEM lanes), B = the (cell, sample) weights
// computed by the CTA's SIMT warps (each weight once per CTA, shared by its 128 channels:
// the paper's component-share principle), D = fp32 accumulators in TMEM.
// Each operand is split x = hi + lo (tc::split_tf32, hi = x rounded to tf32, lo exact); per
// 8-sample K-step one kind::tf32 MMA multiplies the hi parts (exact in fp32) and one kind::f16
// MMA of K = 16 adds both correction terms, bf16(v) bf16(w_lo) + bf16(v_lo) bf16(w_hi)
// (tc::mma8_mix): the fp32 product to <= 2^-17 (RMS 2^-20.6) with 8 MMAs per run (the
// 3xTF32 scheme hi*hi + hi*lo + lo*hi, ~2^-21 with 12 MMAs, with -DHG_TC_MIX=0).
//
// Shared per plan (built on first use, reused by every launch and channel block):
//   * the per-tile chunk schedule {plan position, n, bin row, mask of reachable blocks}
//     (Algorithm 1's "determine the region ... of the contribution points",
//     PAPER.md:209-217, hoisted out of the hot loop);
//   * W per cell, summed by k_tc_wsum from the very same fp32 weights (patch_weights).
//
// k_accum_tc: CTA = 16x12 cells (12 blocks of 4x4) x 128 channels, 512 threads in roles:
//   MMA issuers (warps 0, 3, and 13 with precomputed weights): issuer i issues the MMAs of
//                     the block rows r with r % NI == i: per run of consecutive in-reach
//                     blocks, 4 K-steps x 2 MMAs (N = 16 r), one commit per chunk;
//   warp 1          : value loader: one 2D TMA box (32 plan rows x 128 channels) per chunk
//                     into a 2-stage ring (+ the chunk's geometry in on-the-fly mode);
//   warp 2 (PW)     : weight loader: the chunk's precomputed weight-image bytes into a ring;
//   A producers     : (thread = channel = TMEM lane) split the staged values into the tf32
//                     hi part and the packed bf16 correction operand and tcgen05.st them into
//                     one of 2 TMEM A stages, publishing each chunk before splitting the
//                     next one; every SEG chunks they
//                     add the finished D buffer into the fp32 master tile in shared memory
//                     (D is double-buffered in TMEM, round-to-nearest promotion bounds the
//                     tensor core's truncating accumulation);
//   B producers (OTF): compute the chunk's weights into 2 shared weight stages.
// Epilogue: the last segments are promoted, V = S / W (IEEE div), NaN where W = 0, written as
// coalesced row segments.
// Deterministic: fixed chunk order, fixed work mapping, no atomics.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <type_traits>
#include <vector>

#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "nonfinite.cuh"
#include "weight.cuh"

namespace hg {

// waits of the single-warp roles on the critical hand-off chain (issuers, weight loader)
#ifdef HG_CRIT_SPIN
#define HG_WAIT_CRIT(b, p) tc::mbar_wait_spin((b), (p))
#else
#define HG_WAIT_CRIT(b, p) tc::mbar_wait((b), (p))
#endif

constexpr int TC_THREADS = 512;
constexpr int TC_M = 128;                 // channels per CTA (UMMA M)
#ifndef HG_TC_BY
#define HG_TC_BY 3
#endif
constexpr int TC_BX = 4, TC_BY = HG_TC_BY; // blocks per CTA tile (16 x 4 TC_BY cells)
constexpr int TC_NB = TC_BX * TC_BY;      // 12 blocks
constexpr int TC_N = 16;                  // cells per block: 4 x 4
constexpr int TC_TW = TC_BX * 4, TC_TH = TC_BY * 4;
#ifndef HG_TC_KC
#define HG_TC_KC 32
#endif
constexpr int TC_KC = HG_TC_KC;           // samples per chunk (TC_KC / 8 MMA K-steps)
constexpr int KA = TC_KC / 32;            // 128-B swizzle atoms along K (32 tf32 each)
constexpr int LKA = KA == 2 ? 1 : 0;
static_assert(TC_KC == 32 || TC_KC == 64, "chunks of 32 or 64 samples");
#ifndef HG_TC_NA
#define HG_TC_NA 2
#endif
// NBS = 2 weight stages in the on-the-fly mode.  (Round 1 saw timing-dependent results with
// 3-4 stages before the release-before-consume fix of the shared-stage hand-offs; with the
// fp32 master tile in shared memory, 3 or more stages no longer fit the 227 KB budget, so
// the question is moot for this kernel.  NBS = 2 is bit-deterministic run to run:
// tools/det_otf.sh, profiles/r2/det_otf_nbs.log.)
#ifndef HG_TC_MAXQ
#define HG_TC_MAXQ 8
#endif
#ifndef HG_TC_NBS
#define HG_TC_NBS (HG_TC_MAXQ > 8 ? 1 : 2)
#endif
#ifndef HG_TC_NV
#define HG_TC_NV 2          // 3 measured no faster; its 16 KB go to the weight ring
#endif
#ifndef HG_TC_SEG
#define HG_TC_SEG 8         // segment length for dense plans
#endif
#ifndef HG_TC_SEG_SPARSE
#define HG_TC_SEG_SPARSE 16 // segment length when no block gets more than TC_CPB_SPARSE chunks
#endif
// Mixed-precision products (tc::mma8_mix): per 8-sample K-step one kind::tf32 MMA of
// the hi parts and one kind::f16 (bf16) MMA of K = 16 pairing the two correction terms, 8 MMAs
// per run instead of the 12 of 3xTF32 (HG_TC_MIX=0)
#ifndef HG_TC_MIX
#define HG_TC_MIX 1
#endif
constexpr int NA = HG_TC_NA;              // A stages (TMEM)
constexpr int NBS = HG_TC_NBS;            // B stages (SMEM)
constexpr int NV = HG_TC_NV;              // V staging stages (SMEM)
// max blocks (B slots) per schedule entry (a chunk reaching more gets two entries, 7 % of
// cfg4's chunks).  12 (every block of the tile, one entry per chunk, one 48 KB on-the-fly
// weight stage) measured cfg4 12.89 vs 12.97 ms but cfg3 4.08 vs 3.99 ms and OTF cfg3 8.85 vs
// 8.2 ms, so 8.
constexpr int MAXQ = HG_TC_MAXQ;
// The tensor core's fp32 accumulation truncates, so its error grows with the number of MMAs
// accumulated into one D element.  D is therefore double-buffered in TMEM by segments of
// SEG chunks: while the tensor core accumulates segment s+1 into one buffer, the A warps add
// segment s's buffer into an fp32 master tile in shared memory (round-to-nearest).
constexpr int SEG_DENSE = HG_TC_SEG, SEG_SPARSE = HG_TC_SEG_SPARSE;
// A block touched by at most this many chunks in the whole tile accumulates few enough MMAs
// per segment at SEG_SPARSE (measured: max rel err 4e-6 at cfg4, where the max is 70)
constexpr uint32_t TC_CPB_SPARSE = 80 / KA;
// PW mode (precomputed weight image) from this many 128-channel blocks per launch: measured
// faster than on-the-fly weights even for one block (cfg3 4.7 vs 7.2 ms, cfg2 1.0 vs 1.5 ms),
// so whenever the image fits the memory budget
constexpr unsigned TC_PW_MIN_CBLOCKS = 1;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t D_COLS = TC_NB * TC_N;      // one accumulator buffer: 12 blocks x 16 columns
#ifndef HG_TC_ND
#define HG_TC_ND 2
#endif
constexpr uint32_t A_COL0 = HG_TC_ND * D_COLS;  // 384: A stages after the two D buffers
static_assert(A_COL0 + NA * 2 * TC_KC <= TMEM_COLS, "TMEM budget");
static_assert(SEG_DENSE > NA && SEG_SPARSE > NA, "a segment is promoted NA chunks into the next one");
// B stage layout (per hi / lo half): K-major, 128-byte swizzle.  Row R = 16 q + n (slot q,
// cell n) holds the chunk's 32 tf32 weights (128 B); 8-row groups are 1024-B swizzle atoms
// (SBO = 1024); the 16-B k-quad j of row R sits at chunk position j ^ (R & 7), so the 32
// lanes of a producer warp storing one k-quad each hit 8 distinct bank groups (no
// conflicts); the MMA K-step ks starts 32 B further into the atom.
constexpr uint32_t B_ROW = 128;                      // one swizzle-atom row: 32 tf32
constexpr uint32_t ATOM_SLOT = TC_N * B_ROW;         // 2 KB: one block's 16 cells x 32 samples
constexpr uint32_t B_HALF = MAXQ * KA * ATOM_SLOT;   // 16 KB (32-sample chunks)
constexpr uint32_t B_STAGE = 2 * B_HALF;             // 32 KB (hi + lo)
constexpr int V_ROW = TC_M * 4;                      // 512 B
constexpr int V_STAGE = TC_KC * V_ROW;               // 16 KB
constexpr int W_THREADS = 256;            // B producers (warps 8-15)
constexpr int T_LD = TC_TW * TC_TH + 4;   // epilogue tile row (floats): 16-B aligned, conflict-free
// Chunk completion ring: the issuer commits chunk c's MMAs to done[c % NBF]; every role that
// reuses a resource of chunk c (A stage, B stage, weight-ring bytes) waits on that phase.
constexpr int NBF = 16;
// PW mode (precomputed weight image): the weights of a schedule entry (nq in-reach blocks) are
// nq x 2 KB of tf32 hi then nq x 2 KB of lo, already in the operand layout; one bulk copy per
// entry into a byte ring in shared memory (entries placed contiguously, wrapping to 0).
constexpr uint32_t SLOT_BYTES = KA * ATOM_SLOT;      // one block, one half (hi or lo): 2 KB at K = 32
#ifndef HG_TC_RING_KB
#define HG_TC_RING_KB 94    // as large as the budget allows: cfg4 12.95 / 12.60 ms, cfg3 3.97 / 3.69 ms at 74 / 90 KB
#endif
constexpr uint32_t RING = HG_TC_RING_KB * 1024;
static_assert(RING >= MAXQ * 2 * SLOT_BYTES, "the ring holds the largest entry");
constexpr uint32_t REGION0 = RING > NBS * B_STAGE ? RING : NBS * B_STAGE;

struct TcSmem {
    uint8_t B[REGION0];                   // OTF: NBS weight stages of B_STAGE; PW: the ring
    uint8_t Vs[NV][V_STAGE];
    uint4 Es[NV];                         // the chunk's schedule entry (written by the V loader)
    uint32_t Bmask[NBF];                  // block mask of the chunk in each weight stage / ring entry
    uint32_t Boff[NBF];                   // PW: ring offset of the entry
    long long Wstart[NBF];                // PW weight loader: ring position of each in-flight entry
    // chunk c: A stage c % NA, B stage c % NBS (OTF) or ring entry c % NBF (PW)
    uint64_t a_full[NA], b_full[NBF], done[NBF], v_full[NV], v_empty[NV];
    uint64_t seg_done[2], seg_free[2];    // D buffer d: segment's MMAs complete / promoted
    uint64_t bar_done;
    uint32_t tmem_base;
    alignas(16) float M[TC_M][T_LD];      // fp32 master sums [channel][cell] (padded rows)
};

static_assert(offsetof(TcSmem, B) == 0 && offsetof(TcSmem, Vs) % 1024 == 0, "stage layout");
// Shared memory not worth its own bytes (the weight ring gets them; a larger ring measured
// faster: cfg4 12.95 / 12.85 / 12.60 ms at 74 / 80 / 90 KB):
//  * the chunk's sample geometry (on-the-fly mode only) lives behind the NBS weight stages in
//    the region the ring occupies in the precomputed-weight mode;
static_assert(NBS * B_STAGE + NV * TC_KC * sizeof(float4) <= REGION0, "geometry stages fit behind the B stages");
__device__ __forceinline__ float4* geo_stage(TcSmem& sm, int sv) {
    return reinterpret_cast<float4*>(sm.B + NBS * B_STAGE) + sv * TC_KC;
}
//  * the per-thread dependency sink (see the A producers' release) is the padding column of
//    the master tile (columns TC_TW * TC_TH .. T_LD - 1 are never read);
static_assert((T_LD - TC_TW * TC_TH) * TC_M >= TC_THREADS, "a sink word per thread in the master padding");
__device__ __forceinline__ uint32_t* sink_word(TcSmem& sm, int tid) {
    return reinterpret_cast<uint32_t*>(&sm.M[tid / (T_LD - TC_TW * TC_TH)][TC_TW * TC_TH + tid % (T_LD - TC_TW * TC_TH)]);
}
//  * the tile's W per cell for the epilogue is staged in the ring once every MMA has completed.
static_assert(sizeof(TcSmem) + 1024 <= 232448, "shared memory budget");

// byte offset of (slot q, cell n, sample quad kq) inside one half (hi or lo) of an operand
// with ns slots: K-atom a = kq / 8 holds the ns slots' 16-row groups of that atom
// ([atom][slot][16 rows x 128 B]), so the rows of consecutive slots stay 1024 B per 8 apart
__device__ __forceinline__ uint32_t b_off(int q, int n, int kq, int ns) {
    const int r = q * TC_N + n, a = kq >> 3, k8 = kq & 7;
    return (uint32_t)(a * ns * (int)ATOM_SLOT + (r >> 3) * 1024 + (r & 7) * 128 + ((k8 ^ (r & 7)) << 4));
}

// The B operand of one chunk entry: thread wt (0..255) of the B-producer group computes its
// (sample quad kq, column pair ch2, cell row rr) items of slots q0 = wt >> 6, q0 + 4 (slot q =
// the entry's q-th in-reach block in mask order) and stores them, split into tf32 hi / lo, at
// hi + b_off(q, n, kq) and lo + b_off(q, n, kq).  Used by the on-the-fly B producers (shared
// memory) and by the plan's weight image (global memory): the bytes are identical.
// With HG_TC_MIX the second half holds {bf16(w_lo), bf16(w_hi)} per sample instead of the tf32
// lo part: the operand of the mixed-precision correction MMA (tc::mma8_mix).
__device__ __forceinline__ void entry_weights(const Geom& g, const PlanDev& pd, int i0, int j0,
                                              int wt, const float (&cosr)[TC_BY],
                                              const float4 (&g4)[4], uint32_t pstart, int row,
                                              uint32_t mask, int nq, int ns, uint8_t* hi, uint8_t* lo) {
    const int kq = wt & (8 * KA - 1), ch2 = (wt >> (3 + LKA)) & 1, rr = (wt >> (4 + LKA)) & 3;
    const int q0 = wt >> (6 + LKA);
#pragma unroll 1
    for (int q = q0; q < nq; q += 4 / KA) {
        const int b = (int)__fns(mask, 0, q + 1);      // the q-th set bit of the mask
        const int by = b / TC_BX;
        const int cj = j0 + by * 4 + rr;
        const int ci0 = i0 + (b % TC_BX) * 4;
        float cos_c = cosr[0];
#pragma unroll
        for (int k = 1; k < TC_BY; ++k)
            if (by == k) cos_c = cosr[k];
        float w[4][2];                 // [sample][cell col]
        patch_weights<2>(g, pd, row, cj, ci0, 2 * ch2, cos_c, g4, pstart + 4 * kq, w);
        if (pd.omega) {                // per-sample weights (reading R25): w = omega_n w(d)
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float om = w[u][0] > 0.0f || w[u][1] > 0.0f ? __ldg(&pd.omega[pstart + 4 * kq + u]) : 0.0f;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) w[u][cc] = __fmul_rn(w[u][cc], om);
            }
        }
        if (cj >= g.ny) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) w[u][cc] = 0.0f;
        }
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int n = rr * 4 + 2 * ch2 + cc;
            uint4 h4, l4;
            tc::split_tf32(w[0][cc], h4.x, l4.x);
            tc::split_tf32(w[1][cc], h4.y, l4.y);
            tc::split_tf32(w[2][cc], h4.z, l4.z);
            tc::split_tf32(w[3][cc], h4.w, l4.w);
            if (HG_TC_MIX) {           // {bf16(w_lo), bf16(w_hi)} per sample
                l4.x = tc::pack_bf16(__uint_as_float(l4.x), __uint_as_float(h4.x));
                l4.y = tc::pack_bf16(__uint_as_float(l4.y), __uint_as_float(h4.y));
                l4.z = tc::pack_bf16(__uint_as_float(l4.z), __uint_as_float(h4.z));
                l4.w = tc::pack_bf16(__uint_as_float(l4.w), __uint_as_float(h4.w));
            }
            const uint32_t o = b_off(q, n, kq, ns);
            *reinterpret_cast<uint4*>(hi + o) = h4;
            *reinterpret_cast<uint4*>(lo + o) = l4;
        }
    }
}

// cos(lat) of the cell rows a B-producer thread can touch (rr = its row within a block)
__device__ __forceinline__ void entry_cos_rows(const Geom& g, const PlanDev& pd, int j0, int wt,
                                               float (&cosr)[TC_BY]) {
    const int rr = (wt >> (4 + LKA)) & 3;
#pragma unroll
    for (int by = 0; by < TC_BY; ++by) {
        const int cj = j0 + by * 4 + rr;
        cosr[by] = cj < g.ny ? __ldg(&pd.cos_row[cj]) : 1.0f;
    }
}

// ------------------------------------------------------------------ plan-side pieces
// Can any sample in the chunk's bounding box (cells x in [xlo, xhi], y in [rc-0.5, rc+0.5])
// be within R of any cell of the 4x4 block at (bi, bj)?  Conservative haversine lower
// bound: sin^2(d/2) >= sin^2(dlat_min/2) + cos_min^2 sin^2(dlon_min/2).
__device__ __forceinline__ bool block_reachable(const Geom& g, int bi, int bj, double xlo,
                                                double xhi, int rc) {
    const double dy = fmax(0.0, fmax((double)bj - (rc + 0.5), (rc - 0.5) - (double)(bj + 3)));
    const double dx = fmax(0.0, fmax((double)bi - xhi, xlo - (double)(bi + 3)));
    // latitudes involved: cell rows bj..bj+3 and the sample row extent
    const double y0 = fmin((double)bj, rc - 0.5), y1 = fmax((double)(bj + 3), rc + 0.5);
    const double la = g.crval_lat + (y0 + 1.0 - g.crpix_y) * g.cdelt_lat;
    const double lb = g.crval_lat + (y1 + 1.0 - g.crpix_y) * g.cdelt_lat;
    const double cmin = cos(fmin(89.9, fmax(fabs(la), fabs(lb))) * kDeg2Rad);
    const double sy = sin(0.5 * dy * fabs(g.cdelt_lat) * kDeg2Rad);
    const double sx = sin(0.5 * fmin(dx * fabs(g.cdelt_lon), 180.0) * kDeg2Rad);
    const double hlb = sy * sy + cmin * cmin * sx * sx;
    const double sr = sin(0.5 * g.R_rad);
    return hlb <= sr * sr * (1.0 + 1e-6);
}

// Chunk schedule: one warp per tile; lanes evaluate 32 consecutive chunks of a row at once.
// Entry = {plan position, n | bin row << 8, block mask, 0}.
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
    uint32_t cpb[TC_NB];                    // chunks touching each block (count pass)
#pragma unroll
    for (int b = 0; b < TC_NB; ++b) cpb[b] = 0;
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
                // sample bounding box of the chunk (cell units)
                const double xlo = __float_as_int(pd.geo[p].w) - g.mlon - 0.5;
                const double xhi = __float_as_int(pd.geo[p + n - 1].w) - g.mlon + 0.5;
#pragma unroll
                for (int b = 0; b < TC_NB; ++b) {
                    const int bi = i0 + (b % TC_BX) * 4, bj = j0 + (b / TC_BX) * 4;
                    const bool rows = bj <= rc + g.rl && bj + 3 >= rc - g.rl && bj < g.ny;
                    const bool cols = bi <= chi && bi + 3 >= clo && bi < g.nx;
                    if (rows && cols && block_reachable(g, bi, bj, xlo, xhi, rc)) mk |= 1u << b;
                }
            }
            // entries per chunk: ceil(popc(mask) / MAXQ) (same samples, disjoint block sets)
            const uint32_t ne = (__popc(mk) + MAXQ - 1) / MAXQ;
            uint32_t incl = ne;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            if (n_out) {
#pragma unroll
                for (int b = 0; b < TC_NB; ++b) cpb[b] += __popc(__ballot_sync(0xffffffffu, (mk >> b) & 1u));
                const uint32_t nchunk = __popc(__ballot_sync(0xffffffffu, mk != 0));
                const uint32_t nblk = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mk));
                const uint32_t nsmp = __reduce_add_sync(0xffffffffu, mk ? n : 0u);
                const uint32_t nrun = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mk & ~(mk << 1)));
                const uint32_t nspan = __reduce_add_sync(0xffffffffu, mk ? (uint32_t)(32 - __clz(mk) - __ffs(mk) + 1) : 0u);
                if (lane == 0) {
                    atomicAdd(&n_out[tiles + 1], nchunk);
                    atomicAdd(&n_out[tiles + 2], nblk);
                    atomicAdd(&n_out[tiles + 3], nsmp);
                    atomicAdd(&n_out[tiles + 4], nrun);
                    atomicAdd(&n_out[tiles + 5], nspan);
                }
            }
            if (mk && sched) {
                uint32_t pos = base + cnt + incl - ne;
                uint32_t rest = mk;
                while (rest) {
                    uint32_t part = 0;
                    for (int k = 0; k < MAXQ && rest; ++k) {
                        part |= rest & (~rest + 1u);
                        rest &= rest - 1;
                    }
                    sched[pos++] = make_uint4(p, n | ((uint32_t)br << 8), part, 0u);
                }
            }
            cnt += tot;
        }
    }
    if (n_out && lane == 0) {
        n_out[warp] = cnt;
        uint32_t mx = 0;
#pragma unroll
        for (int b = 0; b < TC_NB; ++b) mx = max(mx, cpb[b]);
        atomicMax(&n_out[tiles], mx);     // max chunks per block over the map
    }
}

// W per cell from the tensor-core engine's own weights (patch_weights), two-level sum
// (per bin row, then compensated) in plan order: deterministic.
__global__ void k_tc_wsum(const __grid_constant__ Geom g, PlanDev pd, float* __restrict__ wsum) {
    const int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (cell >= (int64_t)g.nx * g.ny) return;
    const int i = (int)(cell % g.nx), j = (int)(cell / g.nx);
    const int ci0 = i & ~3, cc = i & 3;
    const float cos_c = pd.cos_row[j];
    float W = 0.0f, Wc = 0.0f;
    for (int br = j; br <= j + 2 * g.mlat; ++br) {
        const int m = pd.mrow[br];
        const int64_t rowb = (int64_t)br * g.ncol;
        const uint32_t s0 = pd.bin_start[rowb + i + g.mlon - m];
        const uint32_t s1 = pd.bin_start[rowb + i + g.mlon + m + 1];
        float part = 0.0f;
        for (uint32_t s = s0; s < s1; s += 4) {
            float4 sv[4];
            const uint32_t nv = min(4u, s1 - s);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                sv[u] = (uint32_t)u < nv ? pd.geo[s + u] : make_float4(0.0f, kInvalidDy, 0.0f, 0.0f);
            }
            float w[4][4];
            patch_weights<4>(g, pd, br, j, ci0, 0, cos_c, sv, s, w);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                part += pd.omega && w[u][cc] > 0.0f ? __fmul_rn(w[u][cc], __ldg(&pd.omega[s + u])) : w[u][cc];
        }
        const float y = part - Wc;
        const float t = W + y;
        Wc = (t - W) - y;
        W = t;
    }
    wsum[cell] = W;
}

// Neighbour export through the tensor-core engine's own pairs: one CTA per tile walks the
// tile's schedule entries and, for every (in-reach block, cell row, sample quad) item,
// computes the 4 x 4 weights with patch_weights -- the expression entry_weights uses for
// the B operand and k_tc_wsum for W -- and emits (cell, original index) for every w > 0 whose
// cell lies in [c0, c1).  A pair the schedule prunes is therefore missing here exactly as it
// is missing from the maps (Algorithm 1's gather set).
// idx == nullptr: count into cnt[cell - c0]; else fill idx[off[cell - c0] + cursor].
__global__ void __launch_bounds__(128)
k_tc_pairs(const __grid_constant__ Geom g, PlanDev pd, const int32_t* __restrict__ perm,
           const uint4* __restrict__ sched, const uint32_t* __restrict__ tile_off, int64_t c0,
           int64_t c1, unsigned long long* __restrict__ cnt, const int64_t* __restrict__ off,
           int64_t* __restrict__ idx) {
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    const int i0 = (blockIdx.x % tiles_x) * TC_TW, j0 = (blockIdx.x / tiles_x) * TC_TH;
    {   // skip tiles with no cell in [c0, c1)
        bool any = false;
        const int i1 = min(i0 + TC_TW, g.nx) - 1;
        for (int j = j0; j < min(j0 + TC_TH, g.ny) && !any; ++j)
            any = (int64_t)j * g.nx + i1 >= c0 && (int64_t)j * g.nx + i0 < c1;
        if (!any) return;
    }
    for (uint32_t ei = tile_off[blockIdx.x]; ei < tile_off[blockIdx.x + 1]; ++ei) {
        const uint4 e = __ldg(&sched[ei]);
        const uint32_t pstart = e.x, nk = e.y & 255;
        const int row = (int)(e.y >> 8), nq = __popc(e.z);
        for (int it = threadIdx.x; it < nq * 4 * (TC_KC / 4); it += blockDim.x) {
            const int kq = it % (TC_KC / 4), rr = (it / (TC_KC / 4)) & 3, q = it / TC_KC;
            const int b = (int)__fns(e.z, 0, q + 1);
            const int cj = j0 + (b / TC_BX) * 4 + rr, ci0 = i0 + (b % TC_BX) * 4;
            if (cj >= g.ny) continue;
            float4 s[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                s[u] = (uint32_t)(4 * kq + u) < nk ? __ldg(&pd.geo[pstart + 4 * kq + u])
                                                  : make_float4(0.0f, kInvalidDy, 0.0f, 0.0f);
            float w[4][4];
            patch_weights<4>(g, pd, row, cj, ci0, 0, __ldg(&pd.cos_row[cj]), s, pstart + 4 * kq, w);
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int64_t cell = (int64_t)cj * g.nx + ci0 + c;
                    if (w[u][c] > 0.0f && cell >= c0 && cell < c1) {
                        const unsigned long long k = atomicAdd(&cnt[cell - c0], 1ull);
                        if (idx) idx[off[cell - c0] + (int64_t)k] = perm[pstart + 4 * kq + u];
                    }
                }
        }
    }
}

// The weight image (PW mode): one CTA of 256 threads per tile walks the tile's entries; the
// threads compute the B-producer items of each entry (entry_weights) into global memory at
// the entry's slots: [nq x 2 KB hi][nq x 2 KB lo], byte-identical to the shared-memory stage.
__global__ void __launch_bounds__(W_THREADS)
k_tc_wimage(const __grid_constant__ Geom g, PlanDev pd, const uint4* __restrict__ sched,
            const uint32_t* __restrict__ tile_off, const uint32_t* __restrict__ wslot,
            uint8_t* __restrict__ wimg) {
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    const int i0 = (blockIdx.x % tiles_x) * TC_TW, j0 = (blockIdx.x / tiles_x) * TC_TH;
    const int wt = threadIdx.x, kq = wt & (8 * KA - 1);
    float cosr[TC_BY];
    entry_cos_rows(g, pd, j0, wt, cosr);
    for (uint32_t ei = tile_off[blockIdx.x]; ei < tile_off[blockIdx.x + 1]; ++ei) {
        const uint4 e = __ldg(&sched[ei]);
        const uint32_t pstart = e.x, nk = e.y & 255;
        const int nq = __popc(e.z);
        float4 g4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            g4[u] = (uint32_t)(4 * kq + u) < nk ? __ldg(&pd.geo[pstart + 4 * kq + u])
                                                : make_float4(0.0f, kInvalidDy, 0.0f, 0.0f);
        uint8_t* hi = wimg + (size_t)__ldg(&wslot[ei]) * (2u * SLOT_BYTES);
        entry_weights(g, pd, i0, j0, wt, cosr, g4, pstart, (int)(e.y >> 8), e.z, nq, nq, hi,
                      hi + (size_t)nq * SLOT_BYTES);
    }
}

// Build the weight image once per plan (first launch that asks for it).  Returns false (and
// leaves the plan in on-the-fly mode) if the image does not fit the memory budget.
// HEGRID_TC_TIMING=1 prints the host-side phases of the one-time per-plan preparation
static void prep_mark(const char* what) {
    static const bool on = getenv("HEGRID_TC_TIMING") != nullptr;
    static auto t0 = std::chrono::steady_clock::now();
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[tc prep] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
}

// The image's size is known from the schedule statistics ((chunk, block) pairs = B slots),
// so the budget check is cheap and a plan whose image did not fit retries on later calls
// (hegrid_opts.weight_image_max_bytes: 0 = 1/4 of the free device memory, > 0 = a byte cap,
// < 0 = never).
static bool ensure_tc_wimage(const hegrid_plan_s* p, cudaStream_t st) {
    if (p->tc_pw == 1) return true;
    const int64_t cap = p->opts.weight_image_max_bytes;
    if (cap < 0) return false;
    const int64_t ne = p->tc_nchunks;
    if (ne <= 0) return false;
    {
        const uint64_t want = (uint64_t)p->tc_stats[1] * 2u * SLOT_BYTES;
        size_t fr = 0, total = 0;
        if (cudaMemGetInfo(&fr, &total) != cudaSuccess) return false;
        if (want > (cap > 0 ? (uint64_t)cap : fr / 4) || want > fr) return false;
    }
    prep_mark("wimage start");
    const Geom& g = p->g;
    const int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    std::vector<uint4> h(ne);
    if (cudaMemcpyAsync(h.data(), p->d_tc_sched, ne * sizeof(uint4), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return false;
    prep_mark("schedule to host");
    std::vector<uint32_t> slot(ne);
    uint64_t tot = 0;
    for (int64_t i = 0; i < ne; ++i) {
        slot[i] = (uint32_t)tot;
        tot += (uint64_t)__builtin_popcount(h[i].z);
    }
    const uint64_t bytes = tot * 2u * SLOT_BYTES;
    if (tot >= (1ull << 32)) return false;
    uint8_t* d_img = nullptr;
    uint32_t* d_slot = nullptr;
    prep_mark("slot scan + meminfo");
    if (plan_alloc(p, &d_img, bytes, st) != cudaSuccess) return false;
    prep_mark("image allocation");
    if (plan_alloc(p, &d_slot, ne * sizeof(uint32_t), st) != cudaSuccess) {
        cudaFreeAsync(d_img, st);
        return false;
    }
    cudaError_t e = cudaMemcpyAsync(d_slot, slot.data(), ne * sizeof(uint32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        k_tc_wimage<<<tiles, W_THREADS, 0, st>>>(g, p->dev(), p->d_tc_sched, p->d_tc_tile_off, d_slot, d_img);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    prep_mark("image kernel");
    if (e != cudaSuccess) {
        cudaFreeAsync(d_img, st);
        cudaFreeAsync(d_slot, st);
        return false;
    }
    p->d_tc_wimg = d_img;
    p->d_tc_wslot = d_slot;
    p->tc_wimg_bytes = (int64_t)bytes;
    p->tc_pw = 1;
    return true;
}

static hegrid_status ensure_tc_plan(const hegrid_plan_s* p, cudaStream_t st) {
    if (p->tc_nchunks >= 0) return HEGRID_OK;
    prep_mark("schedule start");
    const Geom& g = p->g;
    const int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    const int64_t cells = (int64_t)g.nx * g.ny;
    uint32_t* d_n = nullptr;
    float* d_w = nullptr;
    HG_TRY(plan_alloc(p, &d_n, (tiles + 6) * sizeof(uint32_t), st));
    cudaError_t e = plan_alloc(p, &d_w, cells * sizeof(float), st);
    if (e != cudaSuccess) {
        cudaFreeAsync(d_n, st);
        return cuda_status(e);
    }
    const int threads = 128, blocks = (tiles * 32 + threads - 1) / threads;
    e = cudaMemsetAsync(d_n, 0, (tiles + 6) * sizeof(uint32_t), st);
    if (e != cudaSuccess) {
        cudaFreeAsync(d_n, st);
        cudaFreeAsync(d_w, st);
        return cuda_status(e);
    }
    k_tc_schedule<<<blocks, threads, 0, st>>>(g, p->dev(), tiles, d_n, nullptr, nullptr);
    k_tc_wsum<<<(int)((cells + 127) / 128), 128, 0, st>>>(g, p->dev(), d_w);
    count_launch(2);
    std::vector<uint32_t> h(tiles + 6, 0);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d_n, (tiles + 6) * 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFreeAsync(d_n, st);
        cudaFreeAsync(d_w, st);
        return cuda_status(e);
    }
    std::vector<uint32_t> off(tiles + 1, 0);
    for (int t = 0; t < tiles; ++t) off[t + 1] = off[t] + h[t];
    const int64_t total = off[tiles];
    uint4* d_s = nullptr;
    e = plan_alloc(p, &d_s, std::max<int64_t>(total, 1) * sizeof(uint4), st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_n, off.data(), (tiles + 1) * 4, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        k_tc_schedule<<<blocks, threads, 0, st>>>(g, p->dev(), tiles, nullptr, d_n, d_s);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFreeAsync(d_n, st);
        cudaFreeAsync(d_w, st);
        if (d_s) cudaFreeAsync(d_s, st);
        return cuda_status(e);
    }
    prep_mark("schedule + wsum built");
    p->d_tc_sched = d_s;
    p->d_tc_tile_off = d_n;
    p->d_tc_wsum = d_w;
    p->tc_nchunks = total;
    p->tc_max_cpb = h[tiles];
    p->tc_stats[0] = h[tiles + 1];    // chunks (distinct sample groups)
    p->tc_stats[1] = h[tiles + 2];    // (chunk, block) pairs
    p->tc_stats[2] = h[tiles + 3];    // samples over all chunks
    p->tc_stats[3] = h[tiles + 4];    // runs of consecutive blocks
    p->tc_stats[4] = h[tiles + 5];    // block spans
    return HEGRID_OK;
}

// The engine's one-time per-plan tables for launches of n_channels (hegrid_grid builds them
// on the plan's prep stream while its first channel block is in flight).
hegrid_status prepare_tc(const hegrid_plan_s* p, int64_t n_channels_per_launch, cudaStream_t st) {
    HG_TRY_S(ensure_tc_plan(p, st));
    const int ncb = (int)((n_channels_per_launch + TC_M - 1) / TC_M);
    int want_pw = ncb >= (int)TC_PW_MIN_CBLOCKS;
    if (const char* e = getenv("HEGRID_TC_PW")) want_pw = atoi(e);
    if (want_pw) ensure_tc_wimage(p, st);
    return cuda_status(cudaStreamSynchronize(st));
}

// Debug cycle counters (HEGRID_TC_DEBUG bit 32): summed over CTAs.
// 0 total, 1 issuer wait A, 2 issuer wait B, 3 A wait V, 4 A wait A-empty, 5 B wait B-empty,
// 6 V wait V-empty, 7 B work, 8 A work, 9 epilogue, 10 issuer issue
__device__ unsigned long long g_tc_prof[16];
// Timeline of one CTA (profiling builds, HEGRID_TC_DEBUG bit 8192): clock64 per (chunk, event)
__device__ long long g_tl[256][12];
__device__ long long g_tla[256][3][8];   // per A warp: v_full passed, a_full arrive, done passed
#define TL(ev, c) do { if (tl_on && (c) < 256) g_tl[(c)][(ev)] = clock64(); } while (0)

// ------------------------------------------------------------------ the kernel
template <int SEG, bool PW>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_accum_tc(const __grid_constant__ Geom g, const __grid_constant__ CUtensorMap tmap_v,
           PlanDev pd, const uint4* __restrict__ sched,
           const uint32_t* __restrict__ tile_off, const float* __restrict__ wsum,
           const uint8_t* __restrict__ wimg, const uint32_t* __restrict__ wslot,
           int C, int tiles, int cgroup, int super_, int snake, int nsplit,
           float* __restrict__ part, float* __restrict__ out,
           float* __restrict__ wout, NfBuf nf, int dbg_in) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    TcSmem& sm = *reinterpret_cast<TcSmem*>(smem_raw);
    if (tc::smem_u32(smem_raw) & 1023u) __trap();   // swizzle atoms need 1024-B alignment
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // A producers: warps 4-7, plus 8-11 when the weights are precomputed (those warps are the
    // B producers otherwise); each lane quarter's chunk columns are split between its warps
        constexpr int A_WARPS = PW ? 8 : 4, A_GROUPS = A_WARPS / 4, A_THREADS = 32 * A_WARPS;
    constexpr int KPW = TC_KC / A_GROUPS;
#ifndef HG_TC_NI_PW
#define HG_TC_NI_PW 3
#endif
    constexpr int NI = PW ? (TC_BY < HG_TC_NI_PW ? TC_BY : HG_TC_NI_PW) : 2;   // MMA issuer warps
#ifdef HG_TC_PROF
    // debug switches (HEGRID_TC_DEBUG) and cycle counters: only in profiling builds
    const int dbg = dbg_in;
    const bool prof = (dbg & 32) != 0;
#else
    constexpr int dbg = 0;
    constexpr bool prof = false;
    (void)dbg_in;
#endif
    const bool tl_on = prof && (dbg & 8192) && blockIdx.x == 1000;
    const long long t_start = clock64();
    unsigned long long pw[4] = {0, 0, 0, 0};
#define TPROF_BEGIN long long _t0 = prof ? clock64() : 0
#define TPROF_END(k) if (prof) pw[k] += (unsigned long long)(clock64() - _t0)
    const int tiles_x = (g.nx + TC_TW - 1) / TC_TW;
    // CTA -> (tile, channel block): channel blocks in groups of `cgroup`, the group's blocks
    // fastest, so the CTAs resident together share their tiles' weight entries in L2
    int tile, cblk;
    {
        const int ncb = (C + TC_M - 1) / TC_M;
        // few CTAs (few tiles x channel blocks): each tile's entries are split into nsplit
        // contiguous parts run by different CTAs, whose partial sums k_tc_reduce adds up
        const int lin = blockIdx.x / nsplit, grp = lin / (tiles * cgroup), within = lin % (tiles * cgroup);
        const int gsz = min(cgroup, ncb - grp * cgroup);
        const int L = within / gsz;
        cblk = grp * cgroup + within % gsz;
        // tile L of the walk: S x S super-tiles (row-major), row-major inside each, so the
        // tiles resident together are 2-D neighbours and share their candidate samples in L2
        const int S = super_, tiles_y = tiles / tiles_x;
        const int band = L / (S * tiles_x), h = min(S, tiles_y - band * S);
        const int bl = L - band * S * tiles_x, sx = bl / (h * S);
        const int w = min(S, tiles_x - sx * S), local = bl - sx * h * S;
        tile = (band * S + local / w) * tiles_x + sx * S + local % w;
    }
    const int i0 = (tile % tiles_x) * TC_TW, j0 = (tile / tiles_x) * TC_TH;
    const int cb = cblk * TC_M;
    const int sp = blockIdx.x % nsplit;              // part of the tile's entries
    const uint32_t e_all = tile_off[tile + 1] - tile_off[tile];
    const uint32_t e_begin = (uint32_t)((uint64_t)e_all * sp / nsplit);
    const uint4* cs = sched + tile_off[tile] + e_begin;
    const int nchunks = (int)((uint64_t)e_all * (sp + 1) / nsplit - e_begin);
    // Tiles of odd tile rows walk their entries backwards (bottom bin rows first): a tile and
    // the one below it then read the bin rows they share at the same stage of their lifetimes,
    // while both are resident, so the second read hits L2.  The order is fixed per tile.
    const bool rev = (snake != 0) && (((tile / tiles_x) & 1) != 0);
    auto ent = [&](int c) { return rev ? nchunks - 1 - c : c; };
    const int64_t cells = (int64_t)g.nx * g.ny;

    if (warp == 0) tc::tmem_alloc(&sm.tmem_base, TMEM_COLS);
    if (tid == 32) {
        for (int s = 0; s < NA; ++s) tc::mbar_init(&sm.a_full[s], A_WARPS);   // one arrive per warp
        for (int s = 0; s < NBF; ++s) {
            tc::mbar_init(&sm.done[s], NI);           // one commit per issuer
            tc::mbar_init(&sm.b_full[s], PW ? 1 : W_THREADS / 32);   // PW: the weight loader's tx
        }
        for (int s = 0; s < NV; ++s) {
            tc::mbar_init(&sm.v_full[s], 1);
            tc::mbar_init(&sm.v_empty[s], PW ? A_WARPS : A_WARPS + W_THREADS / 32);
        }
        for (int d = 0; d < 2; ++d) {
            tc::mbar_init(&sm.seg_done[d], NI);
            tc::mbar_init(&sm.seg_free[d], A_WARPS);
        }
        tc::mbar_init(&sm.bar_done, NI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    {   // the master sums start at 0
        float4* m4 = reinterpret_cast<float4*>(&sm.M[0][0]);
        for (int e = tid; e < TC_M * T_LD / 4; e += TC_THREADS) m4[e] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = sm.tmem_base;
    if (warp >= 4 && warp < 8) {      // both D buffers start at 0 (every MMA accumulates)
        uint32_t z[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) z[k] = 0u;
#pragma unroll
        for (int c0 = 0; c0 < (int)A_COL0; c0 += 32)
            tc::tmem_st32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, z);
        tc::wait_st();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();

    // D buffer d -> master: this warp's lane quarter (channels), blocks in `mask`; with
    // rezero, the blocks are cleared for the buffer's next segment
    // With 8 A warps (PW), the two warps of a lane quarter take alternate blocks.
    auto promote_buffer = [&](int d, uint32_t mask, bool rezero) {
        const int q4 = warp & 3, row = q4 * 32 + lane, grp = (warp - 4) >> 2;
        float* mrow = &sm.M[row][0];
        if (dbg & 1024) mask = 0;
        for (int i = 0; mask; ++i) {
            const int b = __ffs(mask) - 1;
            mask &= mask - 1;
            if (i % A_GROUPS != grp) continue;
            uint32_t r[16];
            const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)d * D_COLS + (uint32_t)(b * TC_N);
            tc::tmem_ld16(ta, r);
            tc::wait_ld();
            if (rezero) {
                uint32_t z16[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) z16[k] = 0u;
                tc::tmem_st16(ta, z16);
            }
            const int x0 = (b % TC_BX) * 4, y0 = (b / TC_BX) * 4;
#pragma unroll
            for (int cy = 0; cy < 4; ++cy) {
                float4* p4 = reinterpret_cast<float4*>(&mrow[(y0 + cy) * TC_TW + x0]);
                float4 v = *p4;
                v.x += __uint_as_float(r[cy * 4 + 0]);
                v.y += __uint_as_float(r[cy * 4 + 1]);
                v.z += __uint_as_float(r[cy * 4 + 2]);
                v.w += __uint_as_float(r[cy * 4 + 3]);
                *p4 = v;
            }
        }
    };
    // Segment s (chunks [s SEG, (s+1) SEG)) uses D buffer s & 1.  The A warps promote it when
    // they are NA chunks into segment s+1 (the issuer has then issued all of segment s), if
    // that chunk exists; the last one or two segments are promoted after the loop.
    const int nseg = (nchunks + SEG - 1) / SEG;
    auto promoted_in_loop = [&](int s) { return (s + 1) * SEG + NA <= nchunks - 1; };

    // MMA issuers: issuer i (warps 0, 3 and, with precomputed weights, 13 -- on different SM
    // sub-partitions) issues the MMAs of the tile's block rows r with r % NI == i, so the
    // per-MMA issue cost is spread over NI instruction streams.  Each D column block is always
    // fed by the same issuer in chunk order: the accumulation order stays fixed.
        const int issuer = warp == 0 ? 0 : (NI > 1 && warp == 3) ? 1 : (NI > 2 && warp == 13) ? 2 : -1;
    if (issuer >= 0) {
        // ============================ MMA issuer =============================
        // chunk c uses A stage c % NA; the loop is unrolled by NA so the stage (and with it
        // every A operand address) is a compile-time constant in each body
        uint32_t rows = 0;
        for (int b = 0; b < TC_NB; ++b)
            if ((b / TC_BX) % NI == issuer) rows |= 1u << b;
        static_assert(NA == 2 || NA == 4, "issuer unrolled for two or four A stages");
        auto issue = [&](const int c, auto SA_) {
            constexpr int sa = decltype(SA_)::value;
            const int seg = c / SEG, d = seg & 1;
            if (c % SEG == 0) {
                // a new segment accumulates into D buffer d, which the A warps have promoted
                // (segment seg - 2) and zeroed
                if (seg >= 2) {
                    TPROF_BEGIN;
                    HG_WAIT_CRIT(&sm.seg_free[d], ((seg >> 1) - 1) & 1);
                    TPROF_END(3);
                    tc::fence_after_sync();
                }
            }
            const int sb = PW ? c % NBF : c % NBS;
            {
                TPROF_BEGIN;
#ifdef HG_TC_NAMED_AFULL
                // named barrier 1 + sa: the A warps arrive, the issuers sync (≈ 20 cycles per
                // hand-off against ≈ 90 through an mbarrier, tools/handoff_bench.cu)
                asm volatile("bar.sync %0, %1;" :: "r"(1 + sa), "r"(32 * (A_WARPS + NI)) : "memory");
#else
                HG_WAIT_CRIT(&sm.a_full[sa], (c / NA) & 1);
#endif
                TPROF_END(0);
            }
            if (issuer == 0 && lane == 0) TL(3, c);
            {
                TPROF_BEGIN;
                HG_WAIT_CRIT(&sm.b_full[sb], PW ? (c / NBF) & 1 : (c / NBS) & 1);
                TPROF_END(1);
            }
            if (issuer == 0 && lane == 0) TL(4, c);
            tc::fence_after_sync();
            const uint32_t mask = sm.Bmask[sb];
            // B operand: OTF = weight stage sb (lo half at B_HALF); PW = the entry's ring bytes
            // (nq slots of hi, then nq slots of lo)
            const uint32_t b_addr = PW ? tc::smem_u32(&sm.B[sm.Boff[sb]]) : tc::smem_u32(&sm.B[sb * B_STAGE]);
            const int ns = PW ? __popc(mask) : MAXQ;       // slots of the B operand's layout
            const uint64_t lo16 = (uint64_t)((ns * SLOT_BYTES) >> 4);
            TPROF_BEGIN;
            if (!(dbg & 2)) {
                // runs of consecutive in-reach blocks = consecutive B slots (slots follow the
                // mask order); D buffers are zeroed before each segment, so every MMA
                // accumulates.  Each run is 12 MMAs behind one elect.
                const uint32_t dh0 = tc::sdesc_sw128_lo(b_addr);
                const uint32_t a0 = tmem + A_COL0 + sa * 2 * TC_KC;
                const uint32_t dbase = tmem + (uint32_t)d * D_COLS;
                uint32_t mm = mask & rows;
                if (dbg & 65536) {
                    // what-if (profiling builds): one run of N = 16 * ((dbg >> 17) & 15)
                    // cells per entry, issued by issuer 0 (timing only; results garbage)
                    mm = 0;
                    if (issuer == 0) {
                        const int nw = 16 * ((dbg >> 17) & 15);
                        tc::mma12_3xtf32<(32 >> 4), TC_KC>(dbase, a0, dh0, dh0 + (uint32_t)lo16,
                                                           tc::idesc_tf32(TC_M, nw));
                    }
                }
                while (mm) {
                    const int b = __ffs(mm) - 1;
                    const int r = __ffs(~(mm >> b)) - 1;
                    mm &= ~(((1u << r) - 1u) << b);
                    const int q = __popc(mask & ((1u << b) - 1u));     // B slot of block b
#pragma unroll
                    for (int a = 0; a < KA; ++a) {    // K-atom a: K-steps 4a .. 4a + 3
                        const uint32_t bh = dh0 + (uint32_t)(((a * ns + q) * ATOM_SLOT) >> 4);
#if HG_TC_MIX
                        tc::mma8_mix<(32 >> 4), TC_KC>(dbase + (uint32_t)(b * TC_N), a0 + 32 * a, bh,
                                                       bh + (uint32_t)lo16, tc::idesc_tf32(TC_M, TC_N * r),
                                                       tc::idesc_bf16(TC_M, TC_N * r));
#else
                        tc::mma12_3xtf32<(32 >> 4), TC_KC>(dbase + (uint32_t)(b * TC_N), a0 + 32 * a, bh,
                                                           bh + (uint32_t)lo16, tc::idesc_tf32(TC_M, TC_N * r));
#endif
                    }
                }
            }
            if (dbg & 4096) {                          // debug (with no MMAs): plain arrive
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sm.done[c % NBF]);
            } else {
                tc::mma_commit_warp(&sm.done[c % NBF]);    // a commit costs ~100 cycles: one per chunk
            }
            if (c % SEG == SEG - 1 || c == nchunks - 1) tc::mma_commit_warp(&sm.seg_done[d]);
            if (issuer == 0 && lane == 0) TL(5, c);
            __syncwarp();
            TPROF_END(2);
        };
        int c = 0;
        for (; c + NA - 1 < nchunks; c += NA) {
            issue(c, std::integral_constant<int, 0>{});
            issue(c + 1, std::integral_constant<int, 1>{});
            if constexpr (NA == 4) {
                issue(c + 2, std::integral_constant<int, 2>{});
                issue(c + 3, std::integral_constant<int, 3>{});
            }
        }
        if (c < nchunks) issue(c, std::integral_constant<int, 0>{});
        if constexpr (NA == 4) {
            if (c + 1 < nchunks) issue(c + 1, std::integral_constant<int, 1>{});
            if (c + 2 < nchunks) issue(c + 2, std::integral_constant<int, 2>{});
        }
        tc::mma_commit_warp(&sm.bar_done);
        __syncwarp();
    } else if (warp == 1) {
        // ============================ V loader ===============================
        // one 2D TMA box (32 plan rows x 128 channels, out-of-range rows/channels zero) and
        // one bulk copy of the 32 geometry records per chunk, L2 prefetch PF chunks ahead
        // schedule entries: the warp loads 32 at a time (lane l holds entry c0 + l), one
        // batch ahead, and hands each chunk's entry to the consumers through Es[stage]
#ifndef HG_TC_PFX
#define HG_TC_PFX 3
#endif
        constexpr int PF = NV + HG_TC_PFX;
        static_assert(PF < 32, "prefetch distance must stay within the next entry batch");
        auto ld_entry = [&](int c) { return c < nchunks ? __ldg(&cs[ent(c)]) : make_uint4(0, 0, 0, 0); };
        uint4 cur = ld_entry(lane), nxt = ld_entry(32 + lane);
#ifndef HG_TC_NO_VPF
        if (lane == 0)
            for (int c = 0; c < PF && c < nchunks; ++c) tc::tma_prefetch_2d(&tmap_v, cb, (int)__ldg(&cs[ent(c)].x));
#endif
        for (int c = 0; c < nchunks; ++c) {
            if ((c & 31) == 0 && c > 0) {
                cur = nxt;
                nxt = ld_entry(c + 32 + lane);
            }
            uint4 e;
            e.x = __shfl_sync(0xffffffffu, cur.x, c & 31);
            e.y = __shfl_sync(0xffffffffu, cur.y, c & 31);
            e.z = __shfl_sync(0xffffffffu, cur.z, c & 31);
            e.w = __shfl_sync(0xffffffffu, cur.w, c & 31);
            const int cp = c + PF;
            const uint32_t xp = __shfl_sync(0xffffffffu, (cp >> 5) == (c >> 5) ? cur.x : nxt.x, cp & 31);
            {   // the whole warp waits (no single-lane divergent region around the wait: lanes
                // parked at a warp sync slow the other warps of their SM sub-partition); lane 0
                // issues the copies
                const int sv = c % NV;
                if (lane == 0) TL(11, c);
#ifndef HG_TC_NO_VPF
                if (lane == 0 && cp < nchunks) tc::tma_prefetch_2d(&tmap_v, cb, (int)xp);
#endif
                TPROF_BEGIN;
                if (c >= NV) tc::mbar_wait(&sm.v_empty[sv], ((c / NV) - 1) & 1);
                TPROF_END(0);
            }
            if (lane == 0) {
                const uint32_t nk = e.y & 255;
                const int sv = c % NV;
                TL(0, c);
                sm.Es[sv] = e;
                if (dbg & 8) {
                    tc::mbar_arrive(&sm.v_full[sv]);
                } else {
                    // the geometry feeds the on-the-fly B producers only
                    tc::mbar_arrive_expect_tx(&sm.v_full[sv], (uint32_t)V_STAGE + (PW ? 0u : nk * 16));
                    tc::tma_load_2d(&sm.Vs[sv][0], &tmap_v, cb, (int)e.x, &sm.v_full[sv]);
                    if (!PW) tc::bulk_g2s(geo_stage(sm, sv), pd.geo + e.x, nk * 16, &sm.v_full[sv]);
                }
            }
            __syncwarp();
        }
    } else if (PW && warp == 2) {
        // ============================ weight loader (PW) ======================
        // entry c's nq x 4 KB of precomputed weights -> the ring at the next contiguous offset
        // (wrapping to 0); the bytes are reused once every chunk placed there has completed
        // (done[] phases, confirmed in order).  At most NBF entries are in flight.
        // Entry masks and slots are read in groups of G, two groups ahead, into registers
        // (static indices), so no global-load latency sits on the loop.  (An L2 prefetch of
        // the next group's weights, HG_TC_WPF, measured slower: the CTAs of a tile share them.)
        // Every lane runs the loop (identical values; no lanes parked at a warp sync for the
        // whole kernel, measured -2 %), lane 0 issues the stores, arrives and copies.
        const bool wl0 = lane == 0;
        {
            const uint32_t* ws = wslot + tile_off[tile] + e_begin;
            constexpr int G = 8;
            uint32_t zc[G], sc[G], zn[G], sn[G], zf[G], sf[G];
            auto ldg = [&](int g0, uint32_t (&z)[G], uint32_t (&sl)[G]) {
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const int c = g0 + u;
                    z[u] = c < nchunks ? __ldg(&cs[ent(c)].z) : 0u;
                    sl[u] = c < nchunks ? __ldg(&ws[ent(c)]) : 0u;
                }
            };
            auto pf = [&](const uint32_t (&z)[G], const uint32_t (&sl)[G]) {
#ifdef HG_TC_WPF
#pragma unroll
                for (int u = 0; u < G; ++u)
                    if (z[u]) tc::prefetch_l2(wimg + (size_t)sl[u] * (2u * SLOT_BYTES), __popc(z[u]) * 2u * SLOT_BYTES);
#endif
            };
            ldg(0, zc, sc);
            ldg(G, zn, sn);
            ldg(2 * G, zf, sf);
            pf(zc, sc);
            pf(zn, sn);
            long long head = 0;
            long long* starts = sm.Wstart;    // (shared, not a local-memory array)
            int conf = 0;                         // chunks confirmed complete
            for (int g0 = 0; g0 < nchunks; g0 += G) {
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const int c = g0 + u;
                    if (c >= nchunks) break;
#ifdef HG_TC_HALFW
                    const uint32_t bytes = (dbg & 2048) ? 0u : __popc(zc[u]) * 1u * SLOT_BYTES;   // timing experiment
#else
                    const uint32_t bytes = (dbg & 2048) ? 0u : __popc(zc[u]) * 2u * SLOT_BYTES;
#endif
                    long long off = head % RING;
                    if (off + bytes > RING) {
                        head += RING - off;
                        off = 0;
                    }
                    TPROF_BEGIN;
                    // reuse: the slot barrier of chunk c - NBF, and every chunk that started less
                    // than one ring length before this entry's end
                    while (conf < c && (c - conf >= NBF || starts[conf % NBF] < head + (long long)bytes - RING)) {
                        HG_WAIT_CRIT(&sm.done[conf % NBF], (conf / NBF) & 1);
                        ++conf;
                    }
                    TPROF_END(0);
                    const int k = c % NBF;
                    if (wl0) {
                        starts[c % NBF] = head;
                        sm.Bmask[k] = zc[u];
                        sm.Boff[k] = (uint32_t)off;
                        if (dbg & 512) {
                            tc::mbar_arrive(&sm.b_full[k]);
                        } else {
                            TL(7, c);
                            tc::mbar_arrive_expect_tx(&sm.b_full[k], bytes);
                            tc::bulk_g2s(&sm.B[off], wimg + (size_t)sc[u] * (2u * SLOT_BYTES), bytes, &sm.b_full[k]);
                        }
                    }
                    __syncwarp();      // lane 0's starts[] store is seen by the other lanes
                    head += bytes;
                }
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    zc[u] = zn[u];
                    sc[u] = sn[u];
                    zn[u] = zf[u];
                    sn[u] = sf[u];
                }
                ldg(g0 + 3 * G, zf, sf);
                pf(zn, sn);
            }
        }
        __syncwarp();
    }
    // A producers keep the block masks of the (at most two) segments not yet promoted
    uint32_t segmask0 = 0u, segmask1 = 0u;   // (scalars: no local-memory array)
    if (warp >= 4 && warp < 4 + A_WARPS) {
        // ============================ A producers ============================
        // warp (4 + 4 g + q): lane quarter q (TMEM lanes = channels), samples [k0, k0 + KPW)
        const int q4 = warp & 3;
        const int chl = q4 * 32 + lane;            // channel within the block = TMEM lane
        const int k0 = ((warp - 4) >> 2) * KPW;
        // channels >= C arrive as zeros (the tensor map's out-of-range fill)
        const bool ch_ok = !(dbg & 4);
        // Software-pipelined: the values of chunk c+1 are loaded and split while chunk c's
        // tcgen05.st is in flight; chunk c is published (a_full) once its stores completed.
        uint32_t hi[KPW], lo[KPW];
        auto load_split = [&](int c) {
            const int sv = c % NV;
            {
                TPROF_BEGIN;
                tc::mbar_wait(&sm.v_full[sv], (c / NV) & 1);
                TPROF_END(0);
            }
            if (warp == 4 && lane == 0) TL(1, c);
            if (tl_on && lane == 0 && c < 256) g_tla[c][0][warp - 4] = clock64();
            const float* vs = reinterpret_cast<const float*>(&sm.Vs[sv][0]) + k0 * TC_M + chl;
            const uint4 ee = sm.Es[sv];
            const uint32_t nk = ee.y & 255;
            if ((c / SEG) & 1) segmask1 |= ee.z; else segmask0 |= ee.z;
            if (dbg & 256) {                        // debug: no value work
#pragma unroll
                for (int k = 0; k < KPW; ++k) { hi[k] = 0u; lo[k] = 0u; }
            } else if (nk == TC_KC && ch_ok) {     // full chunk: no masking
#pragma unroll
                for (int k = 0; k < KPW; ++k) tc::split_tf32(vs[k * TC_M], hi[k], lo[k]);
            } else {                                // rows >= nk belong to other chunks
#pragma unroll
                for (int k = 0; k < KPW; ++k) {
                    const float v = ((uint32_t)(k0 + k) < nk && ch_ok) ? vs[k * TC_M] : 0.0f;
                    tc::split_tf32(v, hi[k], lo[k]);
                }
            }
            // The values now live in registers: release the value stage (the V loader refills
            // it while this chunk still waits for its A stage).  An mbarrier arrive does not
            // wait for outstanding shared loads, so a store of a value that depends on every
            // loaded word goes first: the sum of the lo parts (lo = v - hi depends on v).
            float s0 = 0.0f, s1 = 0.0f;
#pragma unroll
            for (int k = 0; k < KPW; k += 2) {
                s0 += __uint_as_float(lo[k]);
                s1 += __uint_as_float(lo[k + 1]);
            }
            const float lsum = s0 + s1;
            const uint32_t dep = ee.x ^ ee.y ^ ee.z ^ __float_as_uint(lsum);
            if (warp == 4 && lane == 0 && tl_on && c < 256) g_tl[c][8] = clock64() + (dep == 0x12345u);
            asm volatile("st.shared.u32 [%0], %1;" :: "r"(tc::smem_u32(sink_word(sm, tid))), "r"(dep) : "memory");
            // one arrive per warp (hundreds of per-thread arrives on one mbarrier serialise)
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sm.v_empty[sv]);
            // Non-finite values (nonfinite.cuh): lo is NaN / Inf iff v is non-finite (or
            // beyond the tf32 range), so the same sum flags them.  Such a value is zeroed
            // here -- it cannot poison the block's other cells through 0 * NaN -- and
            // recorded for the fix-up, which applies it to exactly the cells within its
            // support.  (Unrolled: hi / lo must stay in registers.)
            if (nf_bad(lsum)) {
#pragma unroll
                for (int k = 0; k < KPW; ++k) {
                    if (!nf_bad(__uint_as_float(lo[k]))) continue;
                    hi[k] = 0u;
                    lo[k] = 0u;
                    if ((uint32_t)(k0 + k) < nk && cb + chl < C) nf_record(nf, ee.x + k0 + k, cb + chl);
                }
            }
            if constexpr (HG_TC_MIX) {
                // mixed-precision correction operand: {bf16(v), bf16(v_lo)} per sample
#pragma unroll
                for (int k = 0; k < KPW; ++k) {
                    const float l = __uint_as_float(lo[k]);
                    lo[k] = tc::pack_bf16(__uint_as_float(hi[k]) + l, l);
                }
            }
        };
        auto store = [&](int c) {
            const int sa = c % NA;
            {
                TPROF_BEGIN;
                if (c >= NA) tc::mbar_wait(&sm.done[(c - NA) % NBF], ((c - NA) / NBF) & 1);
                TPROF_END(1);
            }
            if (warp == 4 && lane == 0 && c >= NA) TL(6, c - NA);
            if (tl_on && lane == 0 && c >= NA && c - NA < 256) g_tla[c - NA][2][warp - 4] = clock64();
            tc::fence_after_sync();
            const uint32_t ta = tmem + ((uint32_t)(q4 * 32) << 16) + A_COL0 + sa * 2 * TC_KC + k0;
            if (warp == 4 && lane == 0) TL(10, c);
            if (dbg & (256 | 16384)) {
            } else if constexpr (KPW == 64) {
                tc::tmem_st32p(ta, hi);
                tc::tmem_st32p(ta + 32, hi + 32);
                tc::tmem_st32p(ta + TC_KC, lo);
                tc::tmem_st32p(ta + TC_KC + 32, lo + 32);
            } else if constexpr (KPW == 32) {
                tc::tmem_st32(ta, hi);
                tc::tmem_st32(ta + TC_KC, lo);
            } else {
                tc::tmem_st16(ta, hi);
                tc::tmem_st16(ta + TC_KC, lo);
            }
        };
        // promote segment s = cn / SEG - 1 when the A warps are about to store chunk cn =
        // (s + 1) SEG + NA (all of segment s's MMAs were issued: the issuer has consumed
        // chunk cn - NA = (s + 1) SEG)
        auto maybe_promote = [&](int cn) {
            if (cn >= SEG && cn % SEG == NA) {
                const int s = cn / SEG - 1, d = s & 1;
                TPROF_BEGIN;
                tc::mbar_wait(&sm.seg_done[d], (s >> 1) & 1);
                tc::fence_after_sync();
                promote_buffer(d, d ? segmask1 : segmask0, true);
                if (d) segmask1 = 0; else segmask0 = 0;
                tc::wait_st();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sm.seg_free[d]);
                TPROF_END(2);
            }
        };
        auto publish = [&](int c) {
            tc::wait_st();
            if (warp == 4 && lane == 0) TL(9, c);
            tc::fence_before_sync();
#ifdef HG_TC_NAMED_AFULL
            asm volatile("bar.arrive %0, %1;" :: "r"(1 + c % NA), "r"(32 * (A_WARPS + NI)) : "memory");
#else
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sm.a_full[c % NA]);
#endif
            if (warp == 4 && lane == 0) TL(2, c);
            if (tl_on && lane == 0 && c < 256) g_tla[c][1][warp - 4] = clock64();
        };
        // Chunk c is stored and published before chunk c + 1's values are loaded and split:
        // the split runs while chunk c's MMAs execute, off the A -> issuer -> done cycle.
        if (nchunks > 0) load_split(0);
        for (int c = 0; c < nchunks; ++c) {
            maybe_promote(c);
            store(c);
            publish(c);
            if (c + 1 < nchunks) {
                TPROF_BEGIN;
                load_split(c + 1);
                TPROF_END(3);
            }
        }
    } else if (!PW && warp >= 8) {
        // ============================ B producers ============================
        // (on-the-fly mode only) item = (slot q, cell row rr, column pair ch2, sample quad
        // kq): 4 samples x 2 cells; a thread keeps (kq, ch2, rr) and takes slots q0, q0 + 4
        const int wt = tid - 8 * 32;                  // 0..255
        const int kq = wt & (8 * KA - 1);
        float cosr[TC_BY];
        entry_cos_rows(g, pd, j0, wt, cosr);
        for (int c = 0; c < nchunks; ++c) {
            const int sv = c % NV;
            float4 g4[4];
            {
                TPROF_BEGIN;
                tc::mbar_wait(&sm.v_full[sv], (c / NV) & 1);
                TPROF_END(2);
            }
            const uint4 e = sm.Es[sv];
            const uint32_t pstart = e.x, nk = e.y & 255, mask = e.z;
            const int row = (int)(e.y >> 8);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                g4[u] = geo_stage(sm, sv)[4 * kq + u];
                if ((uint32_t)(4 * kq + u) >= nk) g4[u] = make_float4(0.0f, kInvalidDy, 0.0f, 0.0f);
            }
            // Release the value stage now.  An mbarrier arrive does not wait for this
            // thread's outstanding shared loads, so first make an instruction consume every
            // loaded word: a store of their xor (it cannot issue before the loads returned).
            {
                uint32_t dep = e.x ^ e.y ^ e.z ^ e.w;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    dep ^= __float_as_uint(g4[u].x) ^ __float_as_uint(g4[u].y) ^
                           __float_as_uint(g4[u].z) ^ __float_as_uint(g4[u].w);
                asm volatile("st.shared.u32 [%0], %1;" :: "r"(tc::smem_u32(sink_word(sm, tid))), "r"(dep) : "memory");
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sm.v_empty[sv]);
            }

            const int sb = c % NBS;
            {
                TPROF_BEGIN;
                if (c >= NBS) tc::mbar_wait(&sm.done[(c - NBS) % NBF], ((c - NBS) / NBF) & 1);
                TPROF_END(0);
            }
            TPROF_BEGIN;
            const int nq = (dbg & 1) ? 0 : __popc(mask);
            uint8_t* bst = &sm.B[sb * B_STAGE];
            entry_weights(g, pd, i0, j0, wt, cosr, g4, pstart, row, mask, nq, MAXQ, bst, bst + B_HALF);
            if (wt == 0) sm.Bmask[sb] = mask;
            if (!(dbg & 128)) tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&sm.b_full[sb]);
            TPROF_END(1);
        }
    }

    const long long t_loop = clock64();
    __syncthreads();
    // ---- epilogue: promote the segments still in TMEM, then coalesced row segments of the
    // master tile to out: V = S / W (Eq. 1's division), NaN where W = 0
    tc::mbar_wait(&sm.bar_done, 0);
    tc::fence_after_sync();
    if (warp >= 4 && warp < 4 + A_WARPS) {
        for (int s = (nseg >= 2 ? nseg - 2 : 0); s < nseg; ++s)
            if (!promoted_in_loop(s)) promote_buffer(s & 1, (s & 1) ? segmask1 : segmask0, false);
    }
    if (tid < TC_TW * TC_TH) {
        const int i = i0 + tid % TC_TW, j = j0 + tid / TC_TW;
        reinterpret_cast<float*>(sm.B)[tid] = (i < g.nx && j < g.ny) ? __ldg(&wsum[(int64_t)j * g.nx + i]) : 0.0f;
    }
    __syncthreads();
    {
        const float qnan = __int_as_float(0x7fc00000);
        const int x = lane & 15;
#pragma unroll 4
        for (int it = warp; it < TC_M * (TC_TH / 2); it += TC_THREADS / 32) {
            const int row = it / (TC_TH / 2), y = (it % (TC_TH / 2)) * 2 + (lane >> 4);
            const int ch = cb + row, i = i0 + x, j = j0 + y;
            if (ch < C && i < g.nx && j < g.ny) {
                const float S = sm.M[row][y * TC_TW + x];
                if (nsplit > 1) {                      // partial sum of this part
                    part[((int64_t)sp * C + ch) * cells + (int64_t)j * g.nx + i] = S;
                } else {
                    const float W = reinterpret_cast<const float*>(sm.B)[y * TC_TW + x];
                    out[(int64_t)ch * cells + (int64_t)j * g.nx + i] = W > 0.0f ? __fdiv_rn(S, W) : qnan;
                }
            }
        }
    }
    if (cblk == 0 && sp == 0 && wout != nullptr && tid < TC_TW * TC_TH) {
        const int i = i0 + tid % TC_TW, j = j0 + tid / TC_TW;
        if (i < g.nx && j < g.ny) wout[(int64_t)j * g.nx + i] = __ldg(&wsum[(int64_t)j * g.nx + i]);
    }
    if (prof && lane == 0) {
        const long long t_end = clock64();
        if (warp == 0) {
            atomicAdd(&g_tc_prof[0], (unsigned long long)(t_end - t_start));
            atomicAdd(&g_tc_prof[1], pw[0]);
            atomicAdd(&g_tc_prof[2], pw[1]);
            atomicAdd(&g_tc_prof[10], pw[2]);
            atomicAdd(&g_tc_prof[15], pw[3]);
            atomicAdd(&g_tc_prof[9], (unsigned long long)(t_end - t_loop));
        } else if (warp == 4) {
            atomicAdd(&g_tc_prof[3], pw[0]);
            atomicAdd(&g_tc_prof[4], pw[1]);
            atomicAdd(&g_tc_prof[13], pw[2]);
            atomicAdd(&g_tc_prof[14], pw[3]);
        } else if (warp == 8) {
            atomicAdd(&g_tc_prof[5], pw[0]);
            atomicAdd(&g_tc_prof[7], pw[1]);
            atomicAdd(&g_tc_prof[11], pw[2]);
        } else if (warp == 1) {
            atomicAdd(&g_tc_prof[6], pw[0]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, TMEM_COLS);
}

// Split tiles: out = (sum of the parts' partial sums, in part order) / W, NaN where W = 0.
__global__ void k_tc_reduce(const float* __restrict__ part, int nsplit, int64_t n, int64_t cells,
                            const float* __restrict__ wsum, float* __restrict__ out) {
    const float qnan = __int_as_float(0x7fc00000);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const float W = __ldg(&wsum[e % cells]);
        float S = 0.0f;
        for (int k = 0; k < nsplit; ++k) S += __ldg(&part[k * n + e]);
        out[e] = W > 0.0f ? __fdiv_rn(S, W) : qnan;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
static hegrid_status make_value_tmap(CUtensorMap* tm, const float* d_v, int64_t ldv, int C,
                                     int64_t rows) {
    using encode_fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static encode_fn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return HEGRID_ECUDA;
        fn = (encode_fn)f;
    }
    const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)std::max<int64_t>(rows, 1)};
    const cuuint64_t strides[1] = {(cuuint64_t)ldv * 4};
    const cuuint32_t box[2] = {(cuuint32_t)TC_M, (cuuint32_t)TC_KC};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)d_v, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? HEGRID_OK : HEGRID_EINVAL;
}

hegrid_status launch_accumulate_tc(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                   int64_t n_channels, float* d_out, float* d_weight,
                                   cudaStream_t st) {
    if (n_channels <= 0) return HEGRID_OK;
    if (n_channels > (1LL << 30)) return HEGRID_EINVAL;
    HG_TRY_S(ensure_tc_plan(p, st));
    alignas(64) CUtensorMap tmap;
    HG_TRY_S(make_value_tmap(&tmap, d_v, ldv, (int)n_channels, p->n_used));
    const Geom& g = p->g;
    int C = (int)n_channels;
    int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    const int ncb = (C + TC_M - 1) / TC_M;
    // split the tiles' entry lists when the grid would leave SMs idle: about eight waves of
    // CTAs (finer parts balance the uneven per-tile work; cfg3: 14 parts 3.98 ms, 7 parts 4.14,
    // 5 parts 4.30, tools/split_sweep.sh)
    int nsplit = 1;
    {
        int nsm = 148;
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        const int64_t ctas = (int64_t)tiles * ncb;
        if (ctas < 2 * nsm) nsplit = (int)std::min<int64_t>(16, std::max<int64_t>(1, (8 * nsm + ctas - 1) / ctas));
        if (const char* e = getenv("HEGRID_TC_SPLIT")) nsplit = std::max(1, std::min(16, atoi(e)));
    }
    dim3 grid(tiles * ncb * nsplit);
    float* d_part = nullptr;
    if (nsplit > 1)
        HG_TRY(plan_alloc(p, &d_part, (size_t)nsplit * C * (size_t)g.nx * g.ny * sizeof(float), st));
    size_t smem = sizeof(TcSmem);
    int dbg = 0;
    if (const char* e = getenv("HEGRID_TC_DEBUG")) dbg = atoi(e);
    const bool sparse = p->tc_max_cpb <= TC_CPB_SPARSE;
    const int SEG = sparse ? SEG_SPARSE : SEG_DENSE;
    // Precomputed weights (read once per channel block) beat recomputing them in the kernel
    // even for a single block; HEGRID_TC_PW=0/1 forces the choice.
    int want_pw = ncb >= (int)TC_PW_MIN_CBLOCKS;
    if (const char* e = getenv("HEGRID_TC_PW")) want_pw = atoi(e);
    const bool pw = want_pw && ensure_tc_wimage(p, st);
    // CTA walk (DRAM traffic, not time: the kernel does not wait on DRAM; tools/order_sweep.sh,
    // cfg4): with precomputed weights, groups of 8 channel blocks of a tile run together (the
    // tile's weight entries are read ~4x from HBM instead of 32x), tiles in 3 x 3 super-tiles,
    // odd tile rows walking their entries backwards, so tiles resident together share their
    // candidate samples in L2: 34.4 GB per cfg4 launch against 38.1 GB with all 32 channel
    // blocks of a tile together and row-major tiles (75 GB tile-major, group 1).  On-the-fly
    // weights: tile-major.  Few channel blocks (cfg2, cfg3): row-major tiles, measured faster
    // there.  The snake fixes a tile's accumulation order, so it is on for every launch (both
    // weight modes, any channel count: the maps stay bit-identical across channel blockings;
    // neutral in time for cfg2 / cfg3).  HEGRID_TC_GROUP / _SUPER / _SNAKE override.
    int cgroup = pw ? std::min(ncb, 8) : 1;
    if (const char* e = getenv("HEGRID_TC_GROUP")) cgroup = std::max(1, std::min(ncb, atoi(e)));
    int super_ = pw && ncb >= 8 ? 3 : 1, snake = 1;
    if (const char* e = getenv("HEGRID_TC_SUPER")) super_ = std::max(1, atoi(e));
    if (const char* e = getenv("HEGRID_TC_SNAKE")) snake = atoi(e);
    NfBuf nf;
    HG_TRY_S(nonfinite_alloc(p, &nf, st));
    auto kern = pw ? (sparse ? k_accum_tc<SEG_SPARSE, true> : k_accum_tc<SEG_DENSE, true>)
                   : (sparse ? k_accum_tc<SEG_SPARSE, false> : k_accum_tc<SEG_DENSE, false>);
    HG_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, TC_THREADS, smem, st>>>(g, tmap, p->dev(), p->d_tc_sched, p->d_tc_tile_off,
                                         p->d_tc_wsum, p->d_tc_wimg, p->d_tc_wslot, C, tiles, cgroup,
                                         super_, snake, nsplit, d_part, d_out, d_weight, nf, dbg);
    count_launch();
    if (nsplit > 1) {
        const int64_t n = (int64_t)C * g.nx * g.ny;
        k_tc_reduce<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(
            d_part, nsplit, n, (int64_t)g.nx * g.ny, p->d_tc_wsum, d_out);
        count_launch();
        cudaFreeAsync(d_part, st);
    }
    HG_TRY_S(nonfinite_fix(p, d_v, ldv, C, nf, d_out, st));
    if (dbg & 32) {
        unsigned long long h[16];
        cudaStreamSynchronize(st);
        cudaMemcpyFromSymbol(h, g_tc_prof, sizeof(h));
        const double tot = (double)h[0];
        fprintf(stderr, "[tc prof] CTAs %d, cycles/CTA %.0f | issuer: waitA %.2f waitB %.2f issue %.2f | "
                "A: waitV %.2f waitAempty %.2f | B: waitBempty %.2f waitV %.2f work %.2f | V: waitVempty %.2f | "
                "epilogue %.2f | A promote %.2f loadsplit %.2f | issuer wait free %.2f (fractions of CTA time)\n",
                grid.x * grid.y, tot / (grid.x * grid.y), h[1] / tot, h[2] / tot, h[10] / tot,
                h[3] / tot, h[4] / tot, h[5] / tot, h[11] / tot, h[7] / tot, h[6] / tot, h[9] / tot,
                h[13] / tot, h[14] / tot, h[15] / tot);
        fprintf(stderr, "[tc prof] max chunks per block %u, segment %d chunks | entries %lld, chunks %u, "
                "blocks/chunk %.2f, samples/chunk %.1f, runs/chunk %.2f, span/chunk %.2f\n", p->tc_max_cpb, SEG,
                (long long)p->tc_nchunks, p->tc_stats[0], (double)p->tc_stats[1] / p->tc_stats[0],
                (double)p->tc_stats[2] / p->tc_stats[0], (double)p->tc_stats[3] / p->tc_stats[0],
                (double)p->tc_stats[4] / p->tc_stats[0]);
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(g_tc_prof, z, sizeof(z));
        if (dbg & 8192) {
            static long long tl[256][12];
            cudaMemcpyFromSymbol(tl, g_tl, sizeof(tl));
            const long long t0 = tl[40][0];
            fprintf(stderr, "[tc tl] chunk: Vstart vTMA Avfull Asplit Awaitst Aafull Astore | Igota Igotb Icommit Adone Wcopy (cycles rel. to chunk 40 vTMA)\n");
            for (int c = 40; c < 60; ++c)
                fprintf(stderr, "[tc tl] %3d: %7lld %7lld %7lld %7lld %7lld %7lld %7lld | %7lld %7lld %7lld %7lld %7lld\n", c, tl[c][11] - t0, tl[c][0] - t0, tl[c][1] - t0,
                        tl[c][8] - t0, tl[c][9] - t0, tl[c][2] - t0, tl[c][10] - t0, tl[c][3] - t0, tl[c][4] - t0, tl[c][5] - t0, tl[c][6] - t0, tl[c][7] - t0);
            static long long ta[256][3][8];
            cudaMemcpyFromSymbol(ta, g_tla, sizeof(ta));
            for (int c = 40; c < 50; ++c)
                for (int k = 0; k < 3; ++k) {
                    fprintf(stderr, "[tc tla] %3d %s:", c, k == 0 ? "vfull" : k == 1 ? "afull" : "done ");
                    for (int w = 0; w < 8; ++w) fprintf(stderr, " %7lld", ta[c][k][w] ? ta[c][k][w] - t0 : -1);
                    fprintf(stderr, "\n");
                }
        }
    }
    return cuda_status(cudaGetLastError());
}

}  // namespace hg

namespace hg {

// hegrid_neighbours for the tensor-core engine: the CSR of cells [c0, c1) from k_tc_pairs
// (count pass, host scan, fill pass), each cell's list sorted by original index.
hegrid_status tc_neighbours(const hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* offsets,
                            int64_t* idx, cudaStream_t st) {
    const int64_t nc = c1 - c0;
    offsets[0] = 0;
    if (nc == 0) return HEGRID_OK;
    HG_TRY_S(ensure_tc_plan(p, st));
    const Geom& g = p->g;
    const int tiles = ((g.nx + TC_TW - 1) / TC_TW) * ((g.ny + TC_TH - 1) / TC_TH);
    unsigned long long* d_cnt = nullptr;
    int64_t *d_off = nullptr, *d_idx = nullptr;
    std::vector<unsigned long long> h(nc);
    cudaError_t e = cudaMalloc(&d_cnt, nc * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemsetAsync(d_cnt, 0, nc * sizeof(unsigned long long), st);
    if (e == cudaSuccess && p->n_used > 0) {
        k_tc_pairs<<<tiles, 128, 0, st>>>(g, p->dev(), p->d_perm, p->d_tc_sched, p->d_tc_tile_off,
                                          c0, c1, d_cnt, nullptr, nullptr);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d_cnt, nc * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    for (int64_t q = 0; q < nc && e == cudaSuccess; ++q) offsets[q + 1] = offsets[q] + (int64_t)h[q];
    const int64_t tot = offsets[nc];
    if (e == cudaSuccess && idx && tot > 0) {
        e = cudaMalloc(&d_off, nc * sizeof(int64_t));
        if (e == cudaSuccess) e = cudaMalloc(&d_idx, tot * sizeof(int64_t));
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_off, offsets, nc * 8, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(d_cnt, 0, nc * sizeof(unsigned long long), st);
        if (e == cudaSuccess) {
            k_tc_pairs<<<tiles, 128, 0, st>>>(g, p->dev(), p->d_perm, p->d_tc_sched,
                                              p->d_tc_tile_off, c0, c1, d_cnt, d_off, d_idx);
            count_launch();
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(idx, d_idx, tot * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e == cudaSuccess)
            for (int64_t q = 0; q < nc; ++q) std::sort(idx + offsets[q], idx + offsets[q + 1]);
    }
    cudaFree(d_cnt);
    if (d_off) cudaFree(d_off);
    if (d_idx) cudaFree(d_idx);
    return cuda_status(e);
}

}  // namespace hg
