// grid_simt.cu -- accumulate + normalise (Eq. 1 numerator and W; Algorithm 1's
// "Compute the weight sum / weighted value / Normalize the weighted value / Update cell",
// PAPER.md:219-225), FP32 SIMT engine.
//
// Thread organisation (redesign of PAPER.md:232-243 and the gamma reuse of :320-324):
//   CTA  = 8x8 cells x CB = 32*QC channels; 8 warps.
//   warp = a compact 4x2 block of cells (gamma = 8 cells, sharing one candidate lookup)
//          x the CTA's channel block; lane l owns channels cb + QC*l .. +QC-1 and keeps
//          8 x QC fp32 accumulators in registers.
//   For each bin row in reach, the warp walks the row's contiguous candidate range 32
//   samples at a time: lane t computes the 8 weights of sample t (each (cell, sample)
//   weight computed once per channel block and reused by all QC*32 channels),
//   a ballot skips samples outside all 8 supports, and every remaining sample is a
//   rank-1 update acc[8][QC] += w[8] x v[QC] with v a coalesced 16B-per-lane load of
//   the plan-ordered, channel-contiguous value row.
//   Sums run in plan order, per cell, in fp32; W is reduced by a fixed xor-shuffle tree:
//   results are bit-identical run to run and independent of channel blocking/streams.
//   Epilogue: V = S / W (IEEE div.rn), NaN where W = 0, transposed through shared memory
//   so out_map[c][j][i] rows are written as whole 32-byte sectors.
#include "common.cuh"
#include "nonfinite.cuh"
#include "weight.cuh"

namespace hg {

constexpr int SIMT_THREADS = 256;
constexpr int BW = 4, BH = 2;      // cells per warp block
constexpr int TW = 8, TH = 8;      // cells per CTA tile

__device__ __forceinline__ float4 ldg_nc(const float* p) {
    return __ldg(reinterpret_cast<const float4*>(p));
}

// One sample's QC channel values.  Non-finite values (nonfinite.cuh) are zeroed, so they
// cannot reach the warp block's other cells through 0 * NaN, and recorded (plan position
// `pos`, channel c0 + q) for the fix-up; channels >= C are never recorded.
template <int QC>
__device__ __forceinline__ void load_row(const float* p, bool ok, float* v, uint32_t pos, int c0,
                                         int C, NfBuf nf) {
#pragma unroll
    for (int q4 = 0; q4 < QC; q4 += 4) {
        float4 x = ok ? ldg_nc(p + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
        v[q4] = x.x;
        v[q4 + 1] = x.y;
        v[q4 + 2] = x.z;
        v[q4 + 3] = x.w;
    }
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < QC; ++q) s += v[q];
    if (nf_bad(s)) {
#pragma unroll
        for (int q = 0; q < QC; ++q)
            if (nf_bad(v[q])) {
                v[q] = 0.0f;
                if (c0 + q < C) nf_record(nf, pos, (uint32_t)(c0 + q));
            }
    }
}

template <int QC, bool SPLIT>
__global__ void __launch_bounds__(SIMT_THREADS, (QC == 4 && !SPLIT) ? 2 : 1) k_accum_simt(const __grid_constant__ Geom g, PlanDev pd,
                                                             const float* __restrict__ V,
                                                             int64_t ldv, int C,
                                                             float* __restrict__ out,
                                                             float* __restrict__ wout, NfBuf nf) {
    constexpr int CB = 32 * QC;
    constexpr int SO = TW * TH + 1;                 // padded row of the epilogue tile
    __shared__ float4 wbuf[SIMT_THREADS / 32][32][2];
    extern __shared__ float s_out[];                // [CB][SO]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_x = (g.nx + TW - 1) / TW;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int bi0 = tx * TW + (warp & 1) * BW;
    const int bj0 = ty * TH + (warp >> 1) * BH;
    const int cb = blockIdx.y * CB;
    const int c_lane = cb + QC * lane;
    const bool ch_ok = c_lane < C;

    float acc[8][QC];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int q = 0; q < QC; ++q) acc[k][q] = 0.0f;
    float wsum[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) wsum[k] = 0.0f;

    const bool any_cell = bi0 < g.nx && bj0 < g.ny;
    if (any_cell) {
        const int i_hi = min(bi0 + BW - 1, g.nx - 1);
        const int j_hi = min(bj0 + BH - 1, g.ny - 1);
        float cosc[BH];
        bool rok[BH];
#pragma unroll
        for (int r = 0; r < BH; ++r) {
            rok[r] = bj0 + r < g.ny;
            cosc[r] = rok[r] ? pd.cos_row[bj0 + r] : 1.0f;
        }
        bool cok[BW];
#pragma unroll
        for (int c = 0; c < BW; ++c) cok[c] = bi0 + c < g.nx;

        for (int br = bj0; br <= j_hi + 2 * g.mlat; ++br) {
            // SPLIT: per-bin-row partial sums (two-level summation keeps the fp32 rounding
            // of ~1e5-term sums well inside 1e-5)
            float part[SPLIT ? 8 : 1][SPLIT ? QC : 1];
            if constexpr (SPLIT) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int q = 0; q < QC; ++q) part[k][q] = 0.0f;
            }
            const int m = pd.mrow[br];
            const int64_t rowb = (int64_t)br * g.ncol;
            const uint32_t s0 = pd.bin_start[rowb + bi0 + g.mlon - m];
            const uint32_t s1 = pd.bin_start[rowb + i_hi + g.mlon + m + 1];
            for (uint32_t base = s0; base < s1; base += 32) {
                const uint32_t s = base + lane;
                float w[8];
                if (s < s1) {
                    const float4 geo = pd.geo[s];
                    const float om = pd.omega ? __ldg(&pd.omega[s]) : 1.0f;   // reading R25
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int c = k % BW, r = k / BW;
                        w[k] = (cok[c] && rok[r])
                                   ? __fmul_rn(pair_weight(g, pd, bi0 + c, bj0 + r, cosc[r], br, geo, (int)s), om)
                                   : 0.0f;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) w[k] = 0.0f;
                }
                bool nz = false;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    wsum[k] += w[k];
                    nz |= w[k] != 0.0f;
                }
                wbuf[warp][lane][0] = make_float4(w[0], w[1], w[2], w[3]);
                wbuf[warp][lane][1] = make_float4(w[4], w[5], w[6], w[7]);
                uint32_t mask = __ballot_sync(0xffffffffu, nz);
                __syncwarp();
                // software pipeline: the value row of the next active sample is in flight
                // while the rank-1 update of the current one issues
                float vn[QC];
                int tn = -1;
                if (mask) {
                    tn = __ffs(mask) - 1;
                    mask &= mask - 1;
                    load_row<QC>(V + (int64_t)(base + tn) * ldv + c_lane, ch_ok, vn, base + tn, c_lane, C, nf);
                }
                while (tn >= 0) {
                    const int t = tn;
                    float v[QC];
#pragma unroll
                    for (int q = 0; q < QC; ++q) v[q] = vn[q];
                    tn = -1;
                    if (mask) {
                        tn = __ffs(mask) - 1;
                        mask &= mask - 1;
                        load_row<QC>(V + (int64_t)(base + tn) * ldv + c_lane, ch_ok, vn, base + tn, c_lane, C, nf);
                    }
                    const float4 wa = wbuf[warp][t][0], wb = wbuf[warp][t][1];
                    const float ww[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                    for (int k = 0; k < 8; ++k)
#pragma unroll
                        for (int q = 0; q < QC; ++q) {
                            if constexpr (SPLIT)
                                part[k][q] = fmaf(ww[k], v[q], part[k][q]);
                            else
                                acc[k][q] = fmaf(ww[k], v[q], acc[k][q]);
                        }
                }
                __syncwarp();
            }
            if constexpr (SPLIT) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int q = 0; q < QC; ++q) acc[k][q] += part[k][q];
            }
        }
    }
    // W: fixed xor-shuffle tree over lanes (deterministic)
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) wsum[k] += __shfl_xor_sync(0xffffffffu, wsum[k], o);

    // normalise into the shared tile [CB][SO]
    const float qnan = __int_as_float(0x7fc00000);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int cl = (warp >> 1) * BH * TW + (k / BW) * TW + (warp & 1) * BW + (k % BW);
#pragma unroll
        for (int q = 0; q < QC; ++q)
            s_out[(QC * lane + q) * SO + cl] =
                wsum[k] > 0.0f ? __fdiv_rn(acc[k][q], wsum[k]) : qnan;
    }
    if (blockIdx.y == 0 && wout != nullptr && lane < 8) {
        const int i = bi0 + (lane % BW), j = bj0 + (lane / BW);
        float wk = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (k == lane) wk = wsum[k];
        if (i < g.nx && j < g.ny) wout[(int64_t)j * g.nx + i] = wk;
    }
    __syncthreads();
    const int64_t cells = (int64_t)g.nx * g.ny;
    for (int e = threadIdx.x; e < CB * TW * TH; e += SIMT_THREADS) {
        const int cl = e / (TW * TH), cell = e % (TW * TH);
        const int c = cb + cl;
        const int i = tx * TW + (cell % TW), j = ty * TH + (cell / TW);
        if (c < C && i < g.nx && j < g.ny)
            out[(int64_t)c * cells + (int64_t)j * g.nx + i] = s_out[cl * SO + cell];
    }
}

template <int QC, bool SPLIT>
static hegrid_status launch_qc(const hegrid_plan_s* p, const float* d_v, int64_t ldv, int C,
                               float* d_out, float* d_w, cudaStream_t st) {
    const Geom& g = p->g;
    int tiles = ((g.nx + TW - 1) / TW) * ((g.ny + TH - 1) / TH);
    dim3 grid(tiles, (C + 32 * QC - 1) / (32 * QC));
    size_t smem = sizeof(float) * (32 * QC) * (TW * TH + 1);
    HG_TRY(cudaFuncSetAttribute(k_accum_simt<QC, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
    NfBuf nf;
    HG_TRY_S(nonfinite_alloc(p, &nf, st));
    k_accum_simt<QC, SPLIT><<<grid, SIMT_THREADS, smem, st>>>(g, p->dev(), d_v, ldv, C, d_out, d_w, nf);
    count_launch();
    HG_TRY(cudaGetLastError());
    return nonfinite_fix(p, d_v, ldv, C, nf, d_out, st);
}

hegrid_status launch_accumulate_simt(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                     int64_t n_channels, float* d_out, float* d_weight,
                                     cudaStream_t st) {
    if (n_channels <= 0) return HEGRID_OK;
    if (n_channels > (1LL << 30)) return HEGRID_EINVAL;
    int C = (int)n_channels;
    // dense regime (long per-cell sums): two-level summation, 4 channels per lane
    if (p->max_cand > 2048) return launch_qc<4, true>(p, d_v, ldv, C, d_out, d_weight, st);
    return launch_qc<4, false>(p, d_v, ldv, C, d_out, d_weight, st);
}

}  // namespace hg
