// plan.cu -- the spatial index ("LUT") of HEGrid's shared component, on the device.
//
// Paper (Fig. 3 steps 1,2,4): compute each sample's
// pixel index, sort by it (Block Indirect sort, O(N log N)), reorder coordinates, build a
// ring -> pixel -> sample-range lookup table; shared by every channel.  Here (DESIGN.md
// "Plan layer"): map-aligned cell-sized bins instead of HEALPix pixels, a hand-written
// stable LSD radix sort, and a dense bin_start[] table (exclusive scan of the bin
// histogram), so any longitude interval of one bin row is ONE contiguous sample range.
#include <math.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "weight.cuh"

namespace hg {

// ------------------------------------------------------------------ keys (step 1)
__device__ __forceinline__ void sample_frame(const Geom& g, double lon, double lat, double& x,
                                             double& y) {
    x = __dadd_rn(__dadd_rn(wrap180_d(__dadd_rn(lon, -g.crval_lon)) / g.cdelt_lon, g.crpix_x),
                  -1.0);
    y = __dadd_rn(__dadd_rn(__dadd_rn(lat, -g.crval_lat) / g.cdelt_lat, g.crpix_y), -1.0);
}

__global__ void k_keys(const __grid_constant__ Geom g, const double* __restrict__ lon, const double* __restrict__ lat,
                       int64_t n, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                       int* __restrict__ bad) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    double lo = lon[t], la = lat[t];
    uint32_t key = (uint32_t)g.nbins;
    if (!isfinite(lo) || !isfinite(la) || fabs(la) > 90.0) {
        atomicOr(bad, 1);
    } else {
        double x, y;
        sample_frame(g, lo, la, x, y);
        double bx = floor(x + 0.5), by = floor(y + 0.5);
        double br = by + g.mlat, bc = bx + g.mlon;
        if (br >= 0.0 && br < (double)g.nrow && bc >= 0.0 && bc < (double)g.ncol)
            key = (uint32_t)((int64_t)br * g.ncol + (int64_t)bc);
    }
    keys[t] = key;
    vals[t] = (int32_t)t;
}

// ------------------------------------------------------------------ stable LSD radix sort
constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t* __restrict__ keys,
                                                        int64_t n, int shift,
                                                        uint32_t* __restrict__ counts,
                                                        int ntiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int r = 0; r < RS_ITEMS; ++r) {
        int64_t idx = base + r * RS_THREADS + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1u);
    }
    __syncthreads();
    counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Exclusive scan of `total` u32 counts in place, one CTA (counts <= a few million).
__global__ void __launch_bounds__(1024) k_rs_scan(uint32_t* __restrict__ a, int64_t total) {
    __shared__ uint32_t warp_sums[32];
    int tid = threadIdx.x;
    int64_t chunk = (total + 1023) / 1024;
    int64_t b = tid * chunk, e = min(total, b + chunk);
    uint32_t s = 0;
    for (int64_t k = b; k < e; ++k) s += a[k];
    // block exclusive scan of s
    int lane = tid & 31, w = tid >> 5;
    uint32_t v = s;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[w] = v;
    __syncthreads();
    if (w == 0) {
        uint32_t x = warp_sums[lane];
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += u;
        }
        warp_sums[lane] = x;
    }
    __syncthreads();
    uint32_t run = v - s + (w > 0 ? warp_sums[w - 1] : 0u);
    for (int64_t k = b; k < e; ++k) {
        uint32_t c = a[k];
        a[k] = run;
        run += c;
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(
    const uint32_t* __restrict__ kin, const int32_t* __restrict__ vin,
    uint32_t* __restrict__ kout, int32_t* __restrict__ vout, int64_t n, int shift,
    const uint32_t* __restrict__ offsets, int ntiles) {
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_w[RS_THREADS / 32][256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    s_base[tid] = offsets[(int64_t)tid * ntiles + blockIdx.x];
    const uint32_t lt_mask = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * RS_TILE;
    for (int r = 0; r < RS_ITEMS; ++r) {
        int64_t idx = base + r * RS_THREADS + tid;
        bool valid = idx < n;
        uint32_t key = valid ? kin[idx] : 0u;
        uint32_t d = (key >> shift) & 255u;
        for (int k = 0; k < RS_THREADS / 32; ++k) s_w[k][tid] = 0;
        uint32_t tag = valid ? d : (0x100u | (uint32_t)lane);
        uint32_t peers = __match_any_sync(0xffffffffu, tag);
        uint32_t rank = __popc(peers & lt_mask);
        __syncthreads();
        if (valid && rank == 0) s_w[warp][d] = __popc(peers);
        __syncthreads();
        {   // per-digit exclusive prefix over warps, in warp order (stable)
            uint32_t run = s_base[tid];
            for (int k = 0; k < RS_THREADS / 32; ++k) {
                uint32_t c = s_w[k][tid];
                s_w[k][tid] = run;
                run += c;
            }
            s_base[tid] = run;
        }
        __syncthreads();
        if (valid) {
            uint32_t pos = s_w[warp][d] + rank;
            kout[pos] = key;
            vout[pos] = vin[idx];
        }
        __syncthreads();
    }
}

// Sorts (keys, vals) by the low `bits` bits of keys, stably.  Result in the input arrays.
hegrid_status radix_sort_pairs(uint32_t* d_keys, int32_t* d_vals, int64_t n, int bits,
                               cudaStream_t st) {
    if (n <= 1 || bits <= 0) return HEGRID_OK;
    int ntiles = (int)((n + RS_TILE - 1) / RS_TILE);
    int64_t total = 256LL * ntiles;
    uint32_t *k2 = nullptr, *cnt = nullptr;
    int32_t* v2 = nullptr;
    HG_TRY(scratch_alloc(&k2, n * sizeof(uint32_t), st));
    HG_TRY(scratch_alloc(&v2, n * sizeof(int32_t), st));
    HG_TRY(scratch_alloc(&cnt, total * sizeof(uint32_t), st));
    uint32_t *ka = d_keys, *kb = k2;
    int32_t *va = d_vals, *vb = v2;
    int passes = (bits + 7) / 8;
    for (int p = 0; p < passes; ++p) {
        int shift = 8 * p;
        k_rs_hist<<<ntiles, RS_THREADS, 0, st>>>(ka, n, shift, cnt, ntiles);
        k_rs_scan<<<1, 1024, 0, st>>>(cnt, total);
        k_rs_scatter<<<ntiles, RS_THREADS, 0, st>>>(ka, va, kb, vb, n, shift, cnt, ntiles);
        count_launch(3);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != d_keys) {
        HG_TRY(cudaMemcpyAsync(d_keys, ka, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        HG_TRY(cudaMemcpyAsync(d_vals, va, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    }
    HG_TRY(cudaGetLastError());
    HG_TRY(cudaFreeAsync(k2, st));
    HG_TRY(cudaFreeAsync(v2, st));
    HG_TRY(cudaFreeAsync(cnt, st));
    return HEGRID_OK;
}

// ------------------------------------------------------------------ LUT (step 4)
// bin_start[b] = first plan position whose key >= b, b in [0, nbins].
__global__ void k_bin_start(const uint32_t* __restrict__ keys, int64_t n, int64_t nbins,
                            uint32_t* __restrict__ bin_start) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > n) return;
    int64_t lo = (p == 0) ? 0 : (int64_t)keys[p - 1] + 1;
    int64_t hi = (p == n) ? nbins : (int64_t)keys[p];
    for (int64_t b = lo; b <= hi; ++b) bin_start[b] = (uint32_t)p;
}

// ------------------------------------------------------------------ reorder (step 2)
__global__ void k_gather(const __grid_constant__ Geom g, const double* __restrict__ lon, const double* __restrict__ lat,
                         const uint32_t* __restrict__ keys, const int32_t* __restrict__ perm,
                         int64_t n, int32_t* __restrict__ iperm, float4* __restrict__ geo,
                         double2* __restrict__ ll) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    int32_t s = perm[p];
    iperm[s] = (int32_t)p;
    if (keys[p] >= (uint32_t)g.nbins) return;
    double lo = lon[s], la = lat[s];
    double x, y;
    sample_frame(g, lo, la, x, y);
    double bx = floor(x + 0.5), by = floor(y + 0.5);
    float4 q;
    q.x = (float)(x - bx);
    q.y = (float)(y - by);
    q.z = (float)cos(la * kDeg2Rad);
    q.w = __int_as_float((int)(bx + g.mlon));
    geo[p] = q;
    ll[p] = make_double2(lo, la);
}

// One thread per cell: candidate-range length only -> max over cells (kernel selection).
__global__ void k_max_cand(const __grid_constant__ Geom g, PlanDev pd,
                           unsigned long long* __restrict__ mx) {
    int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (cell >= (int64_t)g.nx * g.ny) return;
    int i = (int)(cell % g.nx), j = (int)(cell / g.nx);
    unsigned long long nc = 0;
    for (int br = j; br <= j + 2 * g.mlat; ++br) {
        int m = pd.mrow[br];
        int64_t rowb = (int64_t)br * g.ncol;
        nc += pd.bin_start[rowb + i + g.mlon + m + 1] - pd.bin_start[rowb + i + g.mlon - m];
    }
    atomicMax(mx, nc);
}

// ------------------------------------------------------------------ host: geometry
static hegrid_status make_geom(hegrid_plan_s* p, std::vector<int>& mrow,
                               std::vector<float>& cos_row) {
    const hegrid_map& m = p->map;
    Geom& g = p->g;
    g.nx = m.nx;
    g.ny = m.ny;
    g.crval_lon = m.crval_lon;
    g.crval_lat = m.crval_lat;
    g.crpix_x = m.crpix_x;
    g.crpix_y = m.crpix_y;
    g.cdelt_lon = m.cdelt_lon;
    g.cdelt_lat = m.cdelt_lat;
    double sigma_deg = p->kern.fwhm_deg / (2.0 * sqrt(2.0 * log(2.0)));
    double R_deg = p->kern.support_sigma * sigma_deg;
    if (R_deg > 1.0) return HEGRID_EUNSUPPORTED;
    if (m.projection != HEGRID_PROJ_CAR) return HEGRID_EUNSUPPORTED;   // bins need a lon/lat grid
    g.sigma_rad = sigma_deg * kDeg2Rad;
    g.R_rad = R_deg * kDeg2Rad;
    const double eps = 1e-6;
    double adlat = fabs(m.cdelt_lat), adlon = fabs(m.cdelt_lon);
    g.rl = (int)floor(R_deg / adlat + 0.5 + eps);
    g.mlat = g.rl;
    // latitude extent of cells and of the bin rows
    double lat0 = m.crval_lat + (1.0 - m.crpix_y) * m.cdelt_lat;
    double lat1 = m.crval_lat + ((double)m.ny - m.crpix_y) * m.cdelt_lat;
    double far_cells = std::max(fabs(lat0), fabs(lat1));
    if (far_cells + R_deg >= 89.0) return HEGRID_EUNSUPPORTED;
    g.nrow = m.ny + 2 * g.mlat;
    mrow.assign(g.nrow, 0);
    double Amax = 0;
    for (int br = 0; br < g.nrow; ++br) {
        // samples of bin row br have y in [br - mlat - 0.5, br - mlat + 0.5]
        double ya = br - g.mlat - 0.5, yb = br - g.mlat + 0.5;
        double la = m.crval_lat + (ya + 1.0 - m.crpix_y) * m.cdelt_lat;
        double lb = m.crval_lat + (yb + 1.0 - m.crpix_y) * m.cdelt_lat;
        double df = std::min(std::max(fabs(la), fabs(lb)), far_cells + R_deg);
        double dc = std::min(df + R_deg, 89.5);
        // haversine: sin^2(dlon/2) cos(lat_c) cos(lat_s) <= sin^2(d/2) <= sin^2(R/2)
        double arg = sin(0.5 * R_deg * kDeg2Rad) / sqrt(cos(df * kDeg2Rad) * cos(dc * kDeg2Rad));
        if (arg >= 1.0) return HEGRID_EUNSUPPORTED;
        double A = 2.0 * asin(arg) / kDeg2Rad * (1.0 + 1e-9);
        if (A >= 90.0) return HEGRID_EUNSUPPORTED;
        Amax = std::max(Amax, A);
        mrow[br] = (int)floor(A / adlon + 0.5 + eps);
    }
    // the fp32 hot-path distance keeps sin^2(dlon/2)'s series through b^8 (weight.cuh):
    // accurate to < 6e-7 for half-longitude offsets b <= 0.5 rad; beyond (fields within a
    // degree or two of a pole) the lon/lat bin index is not used
    if (0.5 * Amax * kDeg2Rad > kMaxHalfDlon) return HEGRID_EUNSUPPORTED;
    g.mlon = 0;
    for (int v : mrow) g.mlon = std::max(g.mlon, v);
    // longitude: no wrap ambiguity between the crval frame and the cell frame
    double c0 = fabs((1.0 - m.crpix_x) * m.cdelt_lon);
    double c1 = fabs(((double)m.nx - m.crpix_x) * m.cdelt_lon);
    if (std::max(c0, c1) + Amax + adlon >= 180.0) return HEGRID_EUNSUPPORTED;
    g.ncol = m.nx + 2 * g.mlon;
    g.nbins = (int64_t)g.nrow * g.ncol;
    if (g.nbins >= (1LL << 31) - 2) return HEGRID_EUNSUPPORTED;
    cos_row.resize(m.ny);
    for (int j = 0; j < m.ny; ++j) {
        double latj = m.crval_lat + ((double)j + 1.0 - m.crpix_y) * m.cdelt_lat;
        cos_row[j] = (float)cos(latj * kDeg2Rad);
    }
    g.dlon_rad = (float)(m.cdelt_lon * kDeg2Rad);
    g.dlat_rad = (float)(m.cdelt_lat * kDeg2Rad);
    double R2 = g.R_rad * g.R_rad;
    g.R2_lo = (float)(R2 * (1.0 - 1e-5));
    g.R2_hi = (float)(R2 * (1.0 + 1e-5));
    const double nk2 = -1.0 / (2.0 * g.sigma_rad * g.sigma_rad) / log(2.0);
    g.neg_k2 = (float)nk2;
    g.tK0 = (float)(4.0 * nk2);
    g.tK1 = (float)(4.0 / 3.0 * nk2);
    g.tK2 = (float)(32.0 / 45.0 * nk2);
    g.t_in = (float)(nk2 * R2 * (1.0 - 1e-5));
    g.t_out = (float)(nk2 * R2 * (1.0 + 1e-5));
    g.wexp = p->kern.kind == HEGRID_KERNEL_TOPHAT ? 0.0f : 1.0f;
    return HEGRID_OK;
}

hegrid_status build_plan(hegrid_plan_s* p, const double* d_lon, const double* d_lat,
                         cudaStream_t st) {
    std::vector<int> mrow;
    std::vector<float> cos_row;
    HG_TRY_S(make_geom(p, mrow, cos_row));
    phase_mark("build: geometry");
    const Geom& g = p->g;
    int64_t n = p->n;
    cudaEvent_t e0, e1;
    HG_TRY(cudaEventCreate(&e0));
    HG_TRY(cudaEventCreate(&e1));
    size_t nn = (size_t)std::max<int64_t>(n, 1);
    HG_TRY(plan_alloc(p, &p->d_keys, nn * sizeof(uint32_t), st));
    HG_TRY(plan_alloc(p, &p->d_perm, nn * sizeof(int32_t), st));
    HG_TRY(plan_alloc(p, &p->d_iperm, nn * sizeof(int32_t), st));
    HG_TRY(plan_alloc(p, &p->d_geo, nn * sizeof(float4), st));
    HG_TRY(plan_alloc(p, &p->d_ll, nn * sizeof(double2), st));
    HG_TRY(plan_alloc(p, &p->d_bin_start, (g.nbins + 1) * sizeof(uint32_t), st));
    HG_TRY(plan_alloc(p, &p->d_mrow, g.nrow * sizeof(int), st));
    HG_TRY(plan_alloc(p, &p->d_cos_row, g.ny * sizeof(float), st));
    HG_TRY(cudaMemcpyAsync(p->d_mrow, mrow.data(), g.nrow * sizeof(int), cudaMemcpyHostToDevice, st));
    HG_TRY(cudaMemcpyAsync(p->d_cos_row, cos_row.data(), g.ny * sizeof(float),
                           cudaMemcpyHostToDevice, st));
    phase_mark("build: allocations");
    int* d_bad = nullptr;
    HG_TRY(plan_alloc(p, &d_bad, sizeof(int), st));
    HG_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    // device time of the plan kernels only (allocations above are not part of it)
    HG_TRY(cudaEventRecord(e0, st));
    if (n > 0) {
        int nb = (int)((n + 255) / 256);
        k_keys<<<nb, 256, 0, st>>>(g, d_lon, d_lat, n, p->d_keys, p->d_perm, d_bad);
        count_launch();
        int bits = 0;
        while ((1LL << bits) < g.nbins + 1) ++bits;
        HG_TRY_S(radix_sort_pairs(p->d_keys, p->d_perm, n, bits, st));
        k_gather<<<nb, 256, 0, st>>>(g, d_lon, d_lat, p->d_keys, p->d_perm, n, p->d_iperm,
                                     p->d_geo, p->d_ll);
        count_launch();
    }
    k_bin_start<<<(int)((n + 1 + 255) / 256), 256, 0, st>>>(p->d_keys, n, g.nbins,
                                                            p->d_bin_start);
    count_launch();
    HG_TRY(cudaGetLastError());
    unsigned long long* d_mx = nullptr;
    HG_TRY(plan_alloc(p, &d_mx, sizeof(unsigned long long), st));
    HG_TRY(cudaMemsetAsync(d_mx, 0, sizeof(unsigned long long), st));
    {
        int64_t cells = (int64_t)g.nx * g.ny;
        k_max_cand<<<(int)((cells + 255) / 256), 256, 0, st>>>(g, p->dev(), d_mx);
        count_launch();
    }
    HG_TRY(cudaGetLastError());
    HG_TRY(cudaEventRecord(e1, st));
    unsigned long long mx = 0;
    HG_TRY(cudaMemcpyAsync(&mx, d_mx, sizeof(mx), cudaMemcpyDeviceToHost, st));
    HG_TRY(cudaFreeAsync(d_mx, st));
    int bad = 0;
    uint32_t used = 0;
    HG_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    HG_TRY(cudaMemcpyAsync(&used, p->d_bin_start + g.nbins, sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, st));
    HG_TRY(cudaFreeAsync(d_bad, st));
    phase_mark("build: enqueued");
    HG_TRY(cudaStreamSynchronize(st));
    phase_mark("build: synchronised");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    p->t_plan_ms = ms;
    if (bad) return HEGRID_EDOMAIN;
    p->n_used = used;
    p->max_cand = (int64_t)mx;
    return HEGRID_OK;
}

// ------------------------------------------------------------------ statistics / neighbours
// One thread per cell: candidate-range length and neighbour count.
__global__ void k_cell_counts(const __grid_constant__ Geom g, PlanDev pd, int64_t c0, int64_t c1,
                              int64_t* __restrict__ cand, int64_t* __restrict__ nbr) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= c1 - c0) return;
    int64_t cell = c0 + q;
    int i = (int)(cell % g.nx), j = (int)(cell / g.nx);
    float cos_c = pd.cos_row[j];
    int64_t nc = 0, nn = 0;
    for (int br = j; br <= j + 2 * g.mlat; ++br) {
        int m = pd.mrow[br];
        int64_t rowb = (int64_t)br * g.ncol;
        uint32_t s0 = pd.bin_start[rowb + i + g.mlon - m];
        uint32_t s1 = pd.bin_start[rowb + i + g.mlon + m + 1];
        nc += s1 - s0;
        for (uint32_t s = s0; s < s1; ++s)
            nn += pair_weight(g, pd, i, j, cos_c, br, pd.geo[s], (int)s) > 0.0f ? 1 : 0;
    }
    if (cand) cand[q] = nc;
    if (nbr) nbr[q] = nn;
}

__global__ void k_cell_fill(const __grid_constant__ Geom g, PlanDev pd, const int32_t* __restrict__ perm, int64_t c0,
                            int64_t c1, const int64_t* __restrict__ off,
                            int64_t* __restrict__ idx) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= c1 - c0) return;
    int64_t cell = c0 + q;
    int i = (int)(cell % g.nx), j = (int)(cell / g.nx);
    float cos_c = pd.cos_row[j];
    int64_t k = off[q];
    for (int br = j; br <= j + 2 * g.mlat; ++br) {
        int m = pd.mrow[br];
        int64_t rowb = (int64_t)br * g.ncol;
        uint32_t s0 = pd.bin_start[rowb + i + g.mlon - m];
        uint32_t s1 = pd.bin_start[rowb + i + g.mlon + m + 1];
        for (uint32_t s = s0; s < s1; ++s)
            if (pair_weight(g, pd, i, j, cos_c, br, pd.geo[s], (int)s) > 0.0f)
                idx[k++] = perm[s];
    }
}

hegrid_status plan_pair_stats(hegrid_plan_s* p, cudaStream_t st) {
    int64_t cells = (int64_t)p->g.nx * p->g.ny;
    int64_t *d_c = nullptr, *d_n = nullptr;
    HG_TRY(cudaMalloc(&d_c, cells * sizeof(int64_t)));
    HG_TRY(cudaMalloc(&d_n, cells * sizeof(int64_t)));
    k_cell_counts<<<(int)((cells + 127) / 128), 128, 0, st>>>(p->g, p->dev(), 0, cells, d_c, d_n);
    count_launch();
    std::vector<int64_t> hc(cells), hn(cells);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), d_c, cells * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hn.data(), d_n, cells * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_c);
    cudaFree(d_n);
    HG_TRY(e);
    hegrid_plan_stats& s = p->stats;
    s.n_candidate_pairs = 0;
    s.n_pairs = 0;
    s.nbr_min = cells ? INT32_MAX : 0;
    s.nbr_max = 0;
    for (int64_t q = 0; q < cells; ++q) {
        s.n_candidate_pairs += hc[q];
        s.n_pairs += hn[q];
        s.nbr_min = std::min<int32_t>(s.nbr_min, (int32_t)hn[q]);
        s.nbr_max = std::max<int32_t>(s.nbr_max, (int32_t)hn[q]);
    }
    s.nbr_mean = cells ? (double)s.n_pairs / cells : 0.0;
    return HEGRID_OK;
}

hegrid_status plan_neighbours(hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* offsets,
                              int64_t* idx, cudaStream_t st) {
    int64_t nc = c1 - c0;
    offsets[0] = 0;
    if (nc == 0) return HEGRID_OK;
    int64_t* d_n = nullptr;
    HG_TRY(cudaMalloc(&d_n, (nc + 1) * sizeof(int64_t)));
    int nb = (int)((nc + 127) / 128);
    k_cell_counts<<<nb, 128, 0, st>>>(p->g, p->dev(), c0, c1, nullptr, d_n);
    count_launch();
    std::vector<int64_t> hn(nc);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(hn.data(), d_n, nc * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        cudaFree(d_n);
        return cuda_status(e);
    }
    for (int64_t q = 0; q < nc; ++q) offsets[q + 1] = offsets[q] + hn[q];
    if (!idx) {
        cudaFree(d_n);
        return HEGRID_OK;
    }
    int64_t tot = offsets[nc];
    int64_t* d_idx = nullptr;
    e = cudaMemcpyAsync(d_n, offsets, (nc + 1) * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMalloc(&d_idx, std::max<int64_t>(tot, 1) * 8);
    if (e == cudaSuccess) {
        k_cell_fill<<<nb, 128, 0, st>>>(p->g, p->dev(), p->d_perm, c0, c1, d_n, d_idx);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(idx, d_idx, tot * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_n);
    if (d_idx) cudaFree(d_idx);
    HG_TRY(e);
    for (int64_t q = 0; q < nc; ++q) std::sort(idx + offsets[q], idx + offsets[q + 1]);
    return HEGRID_OK;
}

}  // namespace hg
