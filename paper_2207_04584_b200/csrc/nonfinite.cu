// nonfinite.cu -- the fix-up of non-finite sample values (see nonfinite.cuh).
#include "nonfinite.cuh"
#include "weight.cuh"

namespace hg {

// out <- IEEE combination of the finite partial result `out` and a non-finite term v: NaN
// if either is NaN or they are infinities of opposite sign, else v's infinity.  Commutative
// and associative, applied with CAS: the result does not depend on the record order.
__device__ __forceinline__ void nf_combine(float* a, float v) {
    unsigned int* u = reinterpret_cast<unsigned int*>(a);
    unsigned int old = *u, assumed;
    const float inf = __int_as_float(0x7f800000);
    if (!isnan(v) && !isinf(v)) v = v > 0.0f ? inf : -inf;   // |v| too large for the tf32 split
    do {
        assumed = old;
        const float o = __uint_as_float(assumed);
        float r;
        if (isnan(o) || isnan(v) || (isinf(o) && o != v))
            r = __int_as_float(0x7fc00000);
        else
            r = v;
        const unsigned int rb = __float_as_uint(r);
        if (rb == assumed) break;
        old = atomicCAS(u, assumed, rb);
    } while (old != assumed);
}

// The cells within R of the sample at plan position p (the engines' own predicate:
// patch_weights > 0) receive channel c's non-finite value.
__device__ void nf_apply(const Geom& g, const PlanDev& pd, const uint32_t* __restrict__ keys,
                         uint32_t p, int c, float v, float* __restrict__ out) {
    const uint32_t key = keys[p];
    const int br = (int)(key / (uint32_t)g.ncol), bc = (int)(key % (uint32_t)g.ncol);
    const int m = pd.mrow[br];
    const int64_t cells = (int64_t)g.nx * g.ny;
    const float4 inv = make_float4(0.0f, kInvalidDy, 0.0f, 0.0f);
    const float4 s[4] = {pd.geo[p], inv, inv, inv};
    for (int j = max(0, br - g.mlat - g.rl); j <= min(g.ny - 1, br - g.mlat + g.rl); ++j) {
        const float cos_c = pd.cos_row[j];
        const int i_lo = max(0, bc - g.mlon - m), i_hi = min(g.nx - 1, bc - g.mlon + m);
        for (int ci0 = i_lo & ~3; ci0 <= i_hi; ci0 += 4) {
            float w[4][4];
            patch_weights<4>(g, pd, br, j, ci0, 0, cos_c, s, p, w);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (w[0][k] > 0.0f && ci0 + k >= i_lo && ci0 + k <= i_hi)
                    nf_combine(&out[(int64_t)c * cells + (int64_t)j * g.nx + ci0 + k], v);
        }
    }
}

__global__ void k_nonfinite_fix(const __grid_constant__ Geom g, PlanDev pd,
                                const uint32_t* __restrict__ keys, const float* __restrict__ V,
                                int64_t ldv, int C, int64_t n_used, NfBuf nf,
                                float* __restrict__ out) {
    const uint32_t count = nf.hdr[0], overflow = nf.hdr[1];
    if (count == 0) return;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (!overflow) {
        for (int64_t r = t0; r < (int64_t)min(count, kNfCap); r += stride) {
            const unsigned long long e = nf.rec[r];
            const uint32_t p = (uint32_t)e;
            const int c = (int)(e >> 32);
            nf_apply(g, pd, keys, p, c, V[(int64_t)p * ldv + c], out);
        }
    } else {   // too many records: scan every value
        for (int64_t e = t0; e < n_used * C; e += stride) {
            const int64_t p = e / C;
            const int c = (int)(e % C);
            const float v = V[p * ldv + c];
            if (nf_bad(v)) nf_apply(g, pd, keys, (uint32_t)p, c, v, out);
        }
    }
}

// HEGRID_NONFINITE_MASK: the cells within R of a recorded non-finite value (p, c) get channel
// c's Eq. 1 recomputed over the finite values only (one warp per cell, fp64 sums over the
// cell's candidate ranges with the SIMT engine's pair_weight):
//   V_c = sum_{n: v_cn finite} w v_cn / sum_{n: v_cn finite} w,   NaN if no finite value.
// Records that hit the same (cell, channel) recompute the same value (idempotent writes).
__device__ void nf_mask_cell(const Geom& g, const PlanDev& pd, const float* __restrict__ V,
                             int64_t ldv, int c, int i, int j, float* __restrict__ out, int lane) {
    const float cos_c = pd.cos_row[j];
    double S = 0.0, Wc = 0.0;
    for (int br = j; br <= j + 2 * g.mlat; ++br) {
        const int m = pd.mrow[br];
        const int64_t rowb = (int64_t)br * g.ncol;
        const uint32_t s0 = pd.bin_start[rowb + i + g.mlon - m];
        const uint32_t s1 = pd.bin_start[rowb + i + g.mlon + m + 1];
        for (uint32_t s = s0 + lane; s < s1; s += 32) {
            float w = pair_weight(g, pd, i, j, cos_c, br, pd.geo[s], (int)s);
            if (pd.omega && w > 0.0f) w = __fmul_rn(w, pd.omega[s]);
            if (w > 0.0f) {
                const float v = V[(int64_t)s * ldv + c];
                if (!nf_bad(v)) {
                    S += (double)w * v;
                    Wc += w;
                }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Wc += __shfl_xor_sync(0xffffffffu, Wc, o);
    }
    if (lane == 0) {
        const int64_t cells = (int64_t)g.nx * g.ny;
        out[(int64_t)c * cells + (int64_t)j * g.nx + i] = Wc > 0.0 ? (float)(S / Wc) : __int_as_float(0x7fc00000);
    }
}

// the cells within R of the sample at plan position p (the engines' predicate), one warp each
__device__ void nf_mask_apply(const Geom& g, const PlanDev& pd, const uint32_t* __restrict__ keys,
                              const float* __restrict__ V, int64_t ldv, uint32_t p, int c,
                              float* __restrict__ out, int warp, int nwarps, int lane) {
    const uint32_t key = keys[p];
    const int br = (int)(key / (uint32_t)g.ncol), bc = (int)(key % (uint32_t)g.ncol);
    const int m = pd.mrow[br];
    const int j0 = max(0, br - g.mlat - g.rl), j1 = min(g.ny - 1, br - g.mlat + g.rl);
    const int i0 = max(0, bc - g.mlon - m), i1 = min(g.nx - 1, bc - g.mlon + m);
    const int ni = i1 - i0 + 1;
    if (ni <= 0 || j1 < j0) return;
    for (int q = warp; q < (j1 - j0 + 1) * ni; q += nwarps) {
        const int j = j0 + q / ni, i = i0 + q % ni;
        const float w = pair_weight(g, pd, i, j, pd.cos_row[j], br, pd.geo[p], (int)p);
        if (w > 0.0f) nf_mask_cell(g, pd, V, ldv, c, i, j, out, lane);
    }
}

__global__ void __launch_bounds__(128)
k_nonfinite_mask(const __grid_constant__ Geom g, PlanDev pd, const uint32_t* __restrict__ keys,
                 const float* __restrict__ V, int64_t ldv, int C, int64_t n_used, NfBuf nf,
                 float* __restrict__ out) {
    const uint32_t count = nf.hdr[0], overflow = nf.hdr[1];
    if (count == 0) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (!overflow) {
        for (int64_t r = blockIdx.x; r < (int64_t)min(count, kNfCap); r += gridDim.x) {
            const unsigned long long e = nf.rec[r];
            nf_mask_apply(g, pd, keys, V, ldv, (uint32_t)e, (int)(e >> 32), out, warp, 4, lane);
        }
    } else {   // too many records: scan every value
        for (int64_t e = blockIdx.x; e < n_used * C; e += gridDim.x) {
            const int64_t p = e / C;
            const int c = (int)(e % C);
            if (nf_bad(V[p * ldv + c])) nf_mask_apply(g, pd, keys, V, ldv, (uint32_t)p, c, out, warp, 4, lane);
        }
    }
}

hegrid_status nonfinite_alloc(const hegrid_plan_s* p, NfBuf* nf, cudaStream_t st) {
    void* b = nullptr;
    HG_TRY(plan_alloc(p, &b, 16 + (size_t)kNfCap * 8, st));
    HG_TRY(cudaMemsetAsync(b, 0, 16, st));
    nf->hdr = reinterpret_cast<uint32_t*>(b);
    nf->rec = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(b) + 16);
    return HEGRID_OK;
}

// Enqueue the fix-up after the launch that filled `nf` (it returns at once when nothing
// was recorded), then release the buffer.
hegrid_status nonfinite_fix(const hegrid_plan_s* p, const float* d_v, int64_t ldv, int C, NfBuf nf,
                            float* d_out, cudaStream_t st) {
    if (p->opts.nonfinite == HEGRID_NONFINITE_MASK)
        k_nonfinite_mask<<<4 * 148, 128, 0, st>>>(p->g, p->dev(), p->d_keys, d_v, ldv, C, p->n_used,
                                                  nf, d_out);
    else
        k_nonfinite_fix<<<4 * 148, 128, 0, st>>>(p->g, p->dev(), p->d_keys, d_v, ldv, C, p->n_used,
                                                 nf, d_out);
    count_launch();
    HG_TRY(cudaGetLastError());
    HG_TRY(cudaFreeAsync(nf.hdr, st));
    return HEGRID_OK;
}

}  // namespace hg
