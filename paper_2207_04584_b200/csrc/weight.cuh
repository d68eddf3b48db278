// weight.cuh -- the (cell, sample) kernel weight of Eq. 1 and its support test.
//
// PAPER.md:219-221 (Algorithm 1): "if d(target_cell[], raw_data[i]) <= R: compute weight
// sum, compute weighted value"; w = exp(-d^2 / 2 sigma^2) (readings R1-R5).
//
// Hot path (fp32): the haversine
//     h = sin^2(dlat/2) + cos(lat_c) cos(lat_s) sin^2(dlon/2),   d^2 = 4 asin^2(sqrt h)
// evaluated by series on exact small offsets: dlat/dlon are (integer bin-to-cell offset +
// the sample's fp32 offset from its bin centre) x cdelt, so no large absolute angles are
// ever rounded to fp32.  Near a pole, pairs within R have half-longitude offsets b of up to
// tens of degrees, so sin^2(b) keeps its series up to the b^8 term (sin2_series): the
// truncation 2 b^10 / 14175 is < 6e-7 relative for b <= kMaxHalfDlon = 0.5 rad, which the
// plan enforces (make_geom: EUNSUPPORTED beyond; HEALPix engine territory).  sin^2(dlat/2)
// keeps two terms: dlat <= R <= 1 deg, truncation < 3e-10.  The support test is decided in fp32 outside a +-1e-5 relative guard
// band around R^2 and re-decided inside it by an fp64 haversine on the original fp64
// coordinates, written out without FMA contraction, so the neighbour set is the fp64 one.
#pragma once

#include "common.cuh"

namespace hg {

// sin^2(b) by its Taylor series through b^8 (relative truncation 2 b^8 / 14175: 5.5e-7 at
// b = 0.5 rad).  |b| is clamped to 1.5 rad, below the polynomial's first maximum (b = 1.55),
// so the result stays increasing in |b| and a far pair (beyond any support) never looks near.
__device__ __forceinline__ float sin2_series(float b) {
    b = fminf(fabsf(b), 1.5f);
    const float x = __fmul_rn(b, b);
    float q = fmaf(x, -1.0f / 315.0f, 2.0f / 45.0f);
    q = fmaf(x, q, -1.0f / 3.0f);
    return fmaf(__fmul_rn(x, q), x, x);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ double wrap180_d(double x) {
    double y = fmod(x, 360.0);
    if (y > 180.0) y = __dadd_rn(y, -360.0);
    if (y <= -180.0) y = __dadd_rn(y, 360.0);
    return y;
}

// fp64 support test d <= R for cell (i, j) and a sample at (lon_s, lat_s) degrees.
#ifdef HG_SUPPORT_INLINE
static __device__ __forceinline__
#else
static __device__ __noinline__
#endif
bool support_fp64(const Geom& g, int i, int j, double lon_s,
                                          double lat_s) {
    double lon_c = __dadd_rn(g.crval_lon,
                             __dmul_rn(__dadd_rn(__dadd_rn((double)i, 1.0), -g.crpix_x),
                                       g.cdelt_lon));
    double lat_c = __dadd_rn(g.crval_lat,
                             __dmul_rn(__dadd_rn(__dadd_rn((double)j, 1.0), -g.crpix_y),
                                       g.cdelt_lat));
    double dlon = __dmul_rn(wrap180_d(__dadd_rn(lon_s, -lon_c)), kDeg2Rad);
    double dlat = __dmul_rn(__dadd_rn(lat_s, -lat_c), kDeg2Rad);
    double s1 = sin(__dmul_rn(0.5, dlat));
    double s2 = sin(__dmul_rn(0.5, dlon));
    double cc = __dmul_rn(cos(__dmul_rn(lat_c, kDeg2Rad)), cos(__dmul_rn(lat_s, kDeg2Rad)));
    double h = __dadd_rn(__dmul_rn(s1, s1), __dmul_rn(cc, __dmul_rn(s2, s2)));
    double r = sqrt(h);
    if (r > 1.0) r = 1.0;
    double d = __dmul_rn(2.0, asin(r));
    return d <= g.R_rad;
}

// d^2 (rad^2) from offsets in cells; cc = cos(lat_c) * cos(lat_s).
__device__ __forceinline__ float pair_d2(const Geom& g, float dx_cells, float dy_cells,
                                         float cc) {
    float a = dy_cells * (0.5f * g.dlat_rad);
    float b = dx_cells * (0.5f * g.dlon_rad);
    float a2 = a * a;
    float sa = a2 * (1.0f - a2 * (1.0f / 3.0f));   // sin^2(dlat/2)
    float sb = sin2_series(b);                     // sin^2(dlon/2)
    float h = sa + cc * sb;
    return 4.0f * h * (1.0f + h * ((1.0f / 3.0f) + h * (8.0f / 45.0f)));  // 4 asin^2(sqrt h)
}

// Full weight: returns 0 outside the support.  (i, j) cell; geo = sample's plan data;
// br = the sample's bin row; p = its plan position (for the fp64 recheck).
__device__ __forceinline__ float pair_weight(const Geom& g, const PlanDev& pd, int i, int j,
                                             float cos_c, int br, float4 geo, int p) {
    int bc = __float_as_int(geo.w);
    float dx = (float)(bc - g.mlon - i) + geo.x;
    float dy = (float)(br - g.mlat - j) + geo.y;
    float d2 = pair_d2(g, dx, dy, cos_c * geo.z);
    bool in;
    if (d2 <= g.R2_lo) {
        in = true;
    } else if (d2 > g.R2_hi) {
        in = false;
    } else {
        double2 ll = pd.ll[p];
        in = support_fp64(g, i, j, ll.x, ll.y);
    }
    return in ? ex2_approx(d2 * g.neg_k2 * g.wexp) : 0.0f;
}

// Weights of a 4 x NCOL (sample x cell) patch: samples s[0..3] (plan positions p0..p0+3)
// against the NCOL consecutive cells ci0 + c0 .. ci0 + c0 + NCOL - 1 of cell row cj (ci0 =
// the 4-aligned first column of the cell block, c0 + NCOL <= 4), sharing the per-sample
// terms (sin^2(dlat/2), cos products, lon offset) between the cells.  Same predicate as
// pair_weight (fp32 outside the guard band, fp64 haversine inside; the rare recheck sits
// behind one branch per patch).  Invalid samples must arrive as {0, 1e18, 0, 0} (their d^2
// is clamped to a 1-radian offset, far outside any support: weight 0); cells >= nx get
// weight 0.  Every weight is computed by the same expression whatever NCOL and c0, so the
// tensor-core engine's B producers (4 x 2 patches) and the plan's W kernel (4 x 4) see
// bit-identical weights.  w[u][j] is the weight of sample u and cell column c0 + j.
constexpr float kInvalidDy = 1e18f;
template <int NCOL>
__device__ __forceinline__ void patch_weights(const Geom& g, const PlanDev& pd, int br, int cj,
                                              int ci0, int c0, float cos_c, const float4 (&s)[4],
                                              uint32_t p0, float (&w)[4][NCOL]) {
    // Every operation is an explicitly rounded intrinsic or fmaf: no FMA contraction is left
    // to the compiler, so each instantiation (NCOL, c0, inlining context) produces the same
    // bits for the same (cell, sample) -- the B operand, W and the neighbour export must
    // agree pair by pair (a contraction difference once moved a pair 1.8e-7 outside the guard
    // band in one of them).
    const float hlon = __fmul_rn(0.5f, g.dlon_rad), hlat = __fmul_rn(0.5f, g.dlat_rad);
    const float fy = (float)(br - g.mlat - cj);
    const int ix = -g.mlon - ci0;
    // exponent t = neg_k2 * d^2 with d^2 = 4 asin^2(sqrt h) = h (4 + 4h/3 + 32h^2/45 + ...)
    uint32_t band = 0;      // bit NCOL u + j: pair inside the guard band
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const float a = fminf(fabsf(__fmul_rn(__fadd_rn(fy, s[u].y), hlat)), 1.0f);
        const float a2 = __fmul_rn(a, a);
        const float sa = fmaf(__fmul_rn(a2, -1.0f / 3.0f), a2, a2);
        const float ccs = __fmul_rn(cos_c, s[u].z);
        const float b0 = __fmul_rn(__fadd_rn((float)(__float_as_int(s[u].w) + ix), s[u].x), hlon);
#pragma unroll
        for (int j = 0; j < NCOL; ++j) {
            const float sbv = sin2_series(__fsub_rn(b0, __fmul_rn((float)(c0 + j), hlon)));
            const float h = fmaf(ccs, sbv, sa);
            const float t = __fmul_rn(h, fmaf(h, fmaf(h, g.tK2, g.tK1), g.tK0));
            band |= (uint32_t)((t < g.t_in) & (t >= g.t_out)) << (u * NCOL + j);
            w[u][j] = t >= g.t_out ? ex2_approx(__fmul_rn(t, g.wexp)) : 0.0f;   // band pairs provisionally in
        }
    }
    if (band) {   // rare: decide the guard-band pairs (flagged above) in fp64
        uint32_t kill = 0;
#pragma unroll 1
        for (uint32_t m = band; m; m &= m - 1) {
            const int k = __ffs(m) - 1, u = k / NCOL, cc = c0 + k % NCOL;
            if (ci0 + cc < g.nx) {
                const double2 ll = pd.ll[p0 + u];
                if (!support_fp64(g, ci0 + cc, cj, ll.x, ll.y)) kill |= 1u << k;
            }
        }
#pragma unroll
        for (int k = 0; k < 4 * NCOL; ++k)
            if ((kill >> k) & 1u) w[k / NCOL][k % NCOL] = 0.0f;
    }
    if (ci0 + c0 + NCOL > g.nx) {
#pragma unroll
        for (int j = 0; j < NCOL; ++j)
            if (ci0 + c0 + j >= g.nx)
#pragma unroll
                for (int u = 0; u < 4; ++u) w[u][j] = 0.0f;
    }
}

}  // namespace hg
