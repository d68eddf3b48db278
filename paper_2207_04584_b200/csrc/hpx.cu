// hpx.cu -- the HEALPix-indexed plan and its gather engine: the paper's own LUT (PAPER.md
// 177-192, sec. 3.1.1, Fig. 4/5) and cell update (Algorithm 1), on the GPU.
//
// Plan (steps 1-4 of Fig. 3/5): k_hpx_keys computes every sample's ring-scheme pixel
// (healpix.cuh), the plan's stable radix sort orders the samples by pixel (ties keep the
// original order), k_hpx_gather stores their fp64 coordinates in that order.  The sorted key
// array is the LUT: a pixel interval [p0, p1] of one ring is the contiguous sample range
// [lower_bound(p0), lower_bound(p1 + 1)).
//
// Gather (Algorithm 1): one CTA per (cell, 128-channel block).  Warp 0 walks the rings that
// can reach the cell (ring_above of colatitude +- R, one ring of margin each way), gets each
// ring's 1-2 pixel intervals (hpx::ring_query) and turns them into sample ranges by binary
// search.  The CTA then walks those samples in batches: thread t tests sample t of the batch
// with the fp64 haversine (the oracle's formula) and stores its weight
// w = exp(-d^2 / 2 sigma^2) (tophat: 1) for d <= R, 0 otherwise; every thread (= channel) then
// adds w v into its fp64 sum.  V = S / W in fp64, written as fp32; NaN where W = 0.
// This engine serves the fields the lon/lat bin index does not (polar caps, >= 180 degrees of
// longitude, R > 1 degree) -- it is Algorithm 1 verbatim, not the tensor-core fast path.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "healpix.cuh"

namespace hg {

constexpr int HPX_THREADS = 128;
constexpr int HPX_MAX_RANGES = 256;     // sample ranges gathered per pass (more: next pass)

struct HpxGeom {
    int64_t nside;
    int nx, ny;
    double crval_lon, crval_lat, crpix_x, crpix_y, cdelt_lon, cdelt_lat;
    double R, sigma;      // rad
    int tophat;
    int mask;             // HEGRID_NONFINITE_MASK: non-finite values leave both sums of their channel
    int projection;       // hegrid_projection
};

// Cell centre (hegrid.h, reading R26).  Projected maps: the cell lies at great-circle
// distance rho = atan(r) (TAN) or asin(r) (SIN) from the reference point in the direction of
// position angle pa = atan2(x, y) (east of north); the point at distance rho and bearing pa
// from (lon0, lat0) follows from the spherical law of cosines.
__device__ __forceinline__ void hpx_cell(const HpxGeom& h, int64_t cell, double* lon, double* lat) {
    const int i = (int)(cell % h.nx), j = (int)(cell / h.nx);
    const double x = ((double)i + 1.0 - h.crpix_x) * h.cdelt_lon;
    const double y = ((double)j + 1.0 - h.crpix_y) * h.cdelt_lat;
    if (h.projection == HEGRID_PROJ_CAR) {
        *lon = h.crval_lon + x;
        *lat = h.crval_lat + y;
        return;
    }
    const double r = sqrt(x * x + y * y) * kDeg2Rad;
    const double rho = h.projection == HEGRID_PROJ_TAN ? atan(r) : (r <= 1.0 ? asin(r) : nan(""));
    const double pa = atan2(x, y);
    const double la0 = h.crval_lat * kDeg2Rad;
    double sl = sin(la0) * cos(rho) + cos(la0) * sin(rho) * cos(pa);
    sl = fmin(1.0, fmax(-1.0, sl));
    const double la = asin(sl);
    const double dlo = atan2(sin(pa) * sin(rho) * cos(la0), cos(rho) - sin(la0) * sl);
    *lat = la / kDeg2Rad;
    *lon = h.crval_lon + dlo / kDeg2Rad;
}

__global__ void k_hpx_keys(int64_t nside, const double* __restrict__ lon, const double* __restrict__ lat,
                           int64_t n, uint32_t* __restrict__ keys, int32_t* __restrict__ perm,
                           int* __restrict__ bad) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double lo = lon[k], la = lat[k];
    if (!isfinite(lo) || !isfinite(la) || fabs(la) > 90.0) {
        atomicExch(bad, 1);
        keys[k] = 0;
    } else {
        keys[k] = (uint32_t)hpx::ang2pix_ring(nside, (90.0 - la) * kDeg2Rad, lo * kDeg2Rad);
    }
    perm[k] = (int32_t)k;
}

__global__ void k_hpx_gather(const double* __restrict__ lon, const double* __restrict__ lat,
                             const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ iperm,
                             double2* __restrict__ ll) {
    const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int32_t o = perm[s];
    iperm[o] = (int32_t)s;
    ll[s] = make_double2(lon[o], lat[o]);
}

__device__ __forceinline__ uint32_t lower_bound(const uint32_t* __restrict__ keys, uint32_t n, uint64_t v) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(&keys[mid]) < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// Walk the cell's candidate sample ranges, ring by ring, HPX_MAX_RANGES at a time: fills
// rb/re (shared) with up to HPX_MAX_RANGES ranges starting at ring *ring (warp 0, lane 0 does
// the ring arithmetic; the binary searches run on the lanes).  Returns the range count and
// advances *ring; 0 when the rings are exhausted.
__device__ int hpx_ranges(const HpxGeom& h, const uint32_t* __restrict__ keys, uint32_t n,
                          double theta_c, double phi_c, int* ring, int ring_end, uint32_t* rb,
                          uint32_t* re) {
    const int lane = threadIdx.x & 31;
    const bool pole = theta_c - h.R <= 0.0 || theta_c + h.R >= M_PI;
    int cnt = 0;
    while (*ring <= ring_end && cnt + 2 <= HPX_MAX_RANGES) {
        // up to 16 rings per round: lane l handles ring *ring + (l >> 1), interval l & 1
        const int r = *ring + (lane >> 1);
        int64_t p0[2] = {0, 0}, p1[2] = {-1, -1};
        int nint = 0;
        if (r <= ring_end) nint = hpx::ring_query(h.nside, r, theta_c, phi_c, h.R, pole, p0, p1);
        const int which = lane & 1;
        const bool has = which < nint;
        uint32_t b = 0, e = 0;
        if (has) {
            b = lower_bound(keys, n, (uint64_t)p0[which]);
            e = lower_bound(keys, n, (uint64_t)p1[which] + 1);
        }
        const bool keep = has && e > b;
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        const int rounds = min(16, ring_end - *ring + 1);
        const int need = __popc(m);
        if (cnt + need > HPX_MAX_RANGES) break;     // (cannot happen: need <= 32 < room check)
        if (keep) {
            const int pos = cnt + __popc(m & ((1u << lane) - 1u));
            rb[pos] = b;
            re[pos] = e;
        }
        cnt += need;
        *ring += rounds;
        if (cnt + 32 > HPX_MAX_RANGES) break;
    }
    return cnt;
}

__device__ __forceinline__ void hpx_ring_span(const HpxGeom& h, double theta_c, int* r0, int* r1) {
    const double tlo = fmax(theta_c - h.R, 0.0), thi = fmin(theta_c + h.R, M_PI);
    *r0 = max(1, hpx::ring_above(h.nside, tlo) - 1);
    *r1 = min(hpx::nrings(h.nside), hpx::ring_above(h.nside, thi) + 2);
}

// fp64 haversine distance (rad) between (lon, lat) deg pairs; weight of the pair or -1 if d > R
__device__ __forceinline__ double hpx_weight(const HpxGeom& h, double clon, double clat, double cosc,
                                             double2 s) {
    double dlon = s.x - clon;
    dlon = dlon - 360.0 * floor((dlon + 180.0) / 360.0);   // wrap to [-180, 180)
    const double sdl = sin(0.5 * dlon * kDeg2Rad), sdb = sin(0.5 * (s.y - clat) * kDeg2Rad);
    const double hv = sdb * sdb + cosc * cos(s.y * kDeg2Rad) * sdl * sdl;
    const double d = 2.0 * asin(fmin(1.0, sqrt(hv)));
    if (!(d <= h.R)) return -1.0;
    return h.tophat ? 1.0 : exp(-d * d / (2.0 * h.sigma * h.sigma));
}

__global__ void __launch_bounds__(HPX_THREADS)
k_hpx_grid(const HpxGeom h, const uint32_t* __restrict__ keys, uint32_t n,
           const double2* __restrict__ ll, const float* __restrict__ omega,
           const float* __restrict__ v, int64_t ldv, int C,
           float* __restrict__ out, float* __restrict__ wout) {
    __shared__ uint32_t rb[HPX_MAX_RANGES], re[HPX_MAX_RANGES];
    __shared__ double ws[HPX_THREADS];
    __shared__ uint32_t ss[HPX_THREADS];
    __shared__ int s_cnt, s_ring;
    const int64_t cell = blockIdx.x;
    const int ch = blockIdx.y * HPX_THREADS + threadIdx.x;
    double clon, clat;
    hpx_cell(h, cell, &clon, &clat);
    const double theta_c = (90.0 - clat) * kDeg2Rad, phi_c = clon * kDeg2Rad;
    const double cosc = cos(clat * kDeg2Rad);
    int r0, r1;
    hpx_ring_span(h, theta_c, &r0, &r1);
    if (threadIdx.x == 0) s_ring = r0;
    __syncthreads();
    double S = 0.0, W = 0.0, Wc = 0.0;
    for (;;) {
        if (threadIdx.x < 32) {
            int ring = s_ring;
            const int cnt = hpx_ranges(h, keys, n, theta_c, phi_c, &ring, r1, rb, re);
            if (threadIdx.x == 0) {
                s_cnt = cnt;
                s_ring = ring;
            }
        }
        __syncthreads();
        const int cnt = s_cnt;
        if (cnt == 0 && s_ring > r1) break;
        for (int q = 0; q < cnt; ++q) {
            for (uint32_t b0 = rb[q]; b0 < re[q]; b0 += HPX_THREADS) {
                const uint32_t s = b0 + threadIdx.x;
                double w = -1.0;
                if (s < re[q]) {
                    w = hpx_weight(h, clon, clat, cosc, __ldg(&ll[s]));
                    if (omega && w >= 0.0) w *= (double)__ldg(&omega[s]);   // reading R25
                }
                ws[threadIdx.x] = w;
                ss[threadIdx.x] = s;
                __syncthreads();
                const int m = min(HPX_THREADS, (int)(re[q] - b0));
                for (int k = 0; k < m; ++k) {
                    const double wk = ws[k];
                    if (wk >= 0.0) {
                        W += wk;
                        if (ch < C) {
                            const float vk = __ldg(&v[(int64_t)ss[k] * ldv + ch]);
                            if (!h.mask || isfinite(vk)) {
                                S += wk * (double)vk;
                                Wc += wk;
                            }
                        }
                    }
                }
                __syncthreads();
            }
        }
        if (s_ring > r1) break;
        __syncthreads();
    }
    const int64_t cells = (int64_t)h.nx * h.ny;
    const double Wv = h.mask ? Wc : W;
    if (ch < C) out[(int64_t)ch * cells + cell] = Wv > 0.0 ? (float)(S / Wv) : __int_as_float(0x7fc00000);
    if (wout && blockIdx.y == 0 && threadIdx.x == 0) wout[cell] = (float)W;
}

// pairs of cells [c0, c1): count (idx == nullptr) or fill original sample indices
__global__ void __launch_bounds__(HPX_THREADS)
k_hpx_pairs(const HpxGeom h, const uint32_t* __restrict__ keys, uint32_t n, const double2* __restrict__ ll,
            const int32_t* __restrict__ perm, int64_t c0, int64_t* __restrict__ cand,
            int64_t* __restrict__ cnt, const int64_t* __restrict__ off, int64_t* __restrict__ idx) {
    __shared__ uint32_t rb[HPX_MAX_RANGES], re[HPX_MAX_RANGES];
    __shared__ int s_cnt, s_ring;
    __shared__ unsigned long long s_k, s_cand;
    const int64_t cell = c0 + blockIdx.x;
    double clon, clat;
    hpx_cell(h, cell, &clon, &clat);
    const double theta_c = (90.0 - clat) * kDeg2Rad, phi_c = clon * kDeg2Rad;
    const double cosc = cos(clat * kDeg2Rad);
    int r0, r1;
    hpx_ring_span(h, theta_c, &r0, &r1);
    if (threadIdx.x == 0) {
        s_ring = r0;
        s_k = 0;
        s_cand = 0;
    }
    __syncthreads();
    for (;;) {
        if (threadIdx.x < 32) {
            int ring = s_ring;
            const int c = hpx_ranges(h, keys, n, theta_c, phi_c, &ring, r1, rb, re);
            if (threadIdx.x == 0) {
                s_cnt = c;
                s_ring = ring;
            }
        }
        __syncthreads();
        const int c = s_cnt;
        for (int q = 0; q < c; ++q) {
            if (threadIdx.x == 0) atomicAdd(&s_cand, (unsigned long long)(re[q] - rb[q]));
            for (uint32_t s = rb[q] + threadIdx.x; s < re[q]; s += HPX_THREADS) {
                if (hpx_weight(h, clon, clat, cosc, __ldg(&ll[s])) >= 0.0) {
                    const unsigned long long k = atomicAdd(&s_k, 1ull);
                    if (idx) idx[off[blockIdx.x] + (int64_t)k] = perm[s];
                }
            }
        }
        __syncthreads();
        if (s_ring > r1) break;
    }
    if (threadIdx.x == 0) {
        if (cnt) cnt[blockIdx.x] = (int64_t)s_k;
        if (cand) cand[blockIdx.x] = (int64_t)s_cand;
    }
}

static HpxGeom hpx_geom(const hegrid_plan_s* p) {
    HpxGeom h;
    h.nside = p->hpx_nside;
    h.nx = p->map.nx;
    h.ny = p->map.ny;
    h.crval_lon = p->map.crval_lon;
    h.crval_lat = p->map.crval_lat;
    h.crpix_x = p->map.crpix_x;
    h.crpix_y = p->map.crpix_y;
    h.cdelt_lon = p->map.cdelt_lon;
    h.cdelt_lat = p->map.cdelt_lat;
    h.sigma = p->kern.fwhm_deg / (2.0 * sqrt(2.0 * log(2.0))) * kDeg2Rad;
    h.R = p->kern.support_sigma * h.sigma;
    h.tophat = p->kern.kind == HEGRID_KERNEL_TOPHAT;
    h.mask = p->opts.nonfinite == HEGRID_NONFINITE_MASK;
    h.projection = p->map.projection;
    return h;
}

hegrid_status build_plan_hpx(hegrid_plan_s* p, const double* d_lon, const double* d_lat,
                             cudaStream_t st) {
    const double sigma = p->kern.fwhm_deg / (2.0 * sqrt(2.0 * log(2.0)));
    const double R = p->kern.support_sigma * sigma;
    const double cell = std::min(fabs(p->map.cdelt_lon), fabs(p->map.cdelt_lat));
    p->hpx_nside = hpx::choose_nside(0.5 * std::min(cell, R) * kDeg2Rad);
    p->g.nx = p->map.nx;
    p->g.ny = p->map.ny;
    p->g.sigma_rad = sigma * kDeg2Rad;
    p->g.R_rad = R * kDeg2Rad;
    const int64_t n = p->n;
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    HG_TRY(plan_alloc(p, &p->d_keys, nn * sizeof(uint32_t), st));
    HG_TRY(plan_alloc(p, &p->d_perm, nn * sizeof(int32_t), st));
    HG_TRY(plan_alloc(p, &p->d_iperm, nn * sizeof(int32_t), st));
    HG_TRY(plan_alloc(p, &p->d_ll, nn * sizeof(double2), st));
    int* d_bad = nullptr;
    HG_TRY(plan_alloc(p, &d_bad, sizeof(int), st));
    HG_TRY(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    cudaEvent_t e0, e1;
    HG_TRY(cudaEventCreate(&e0));
    HG_TRY(cudaEventCreate(&e1));
    HG_TRY(cudaEventRecord(e0, st));
    if (n > 0) {
        const int nb = (int)((n + 255) / 256);
        k_hpx_keys<<<nb, 256, 0, st>>>(p->hpx_nside, d_lon, d_lat, n, p->d_keys, p->d_perm, d_bad);
        count_launch();
        int bits = 0;
        while ((1LL << bits) < hpx::npix(p->hpx_nside)) ++bits;
        HG_TRY_S(radix_sort_pairs(p->d_keys, p->d_perm, n, bits, st));
        k_hpx_gather<<<nb, 256, 0, st>>>(d_lon, d_lat, p->d_perm, n, p->d_iperm, p->d_ll);
        count_launch();
    }
    HG_TRY(cudaGetLastError());
    HG_TRY(cudaEventRecord(e1, st));
    int bad = 0;
    HG_TRY(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    HG_TRY(cudaFreeAsync(d_bad, st));
    HG_TRY(cudaStreamSynchronize(st));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    p->t_plan_ms = ms;
    if (bad) return HEGRID_EDOMAIN;
    p->n_used = n;
    return HEGRID_OK;
}

hegrid_status launch_accumulate_hpx(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                    int64_t n_channels, float* d_out, float* d_weight,
                                    cudaStream_t st) {
    const int64_t cells = (int64_t)p->map.nx * p->map.ny;
    if (cells == 0 || n_channels <= 0) return HEGRID_OK;
    if (n_channels > (1LL << 30) || cells > (1LL << 31) - 1) return HEGRID_EINVAL;
    const dim3 grid((unsigned)cells, (unsigned)((n_channels + HPX_THREADS - 1) / HPX_THREADS));
    if (grid.y > 65535) return HEGRID_EINVAL;
    k_hpx_grid<<<grid, HPX_THREADS, 0, st>>>(hpx_geom(p), p->d_keys, (uint32_t)p->n_used, p->d_ll,
                                             p->d_omega, d_v, ldv, (int)n_channels, d_out, d_weight);
    count_launch();
    return cuda_status(cudaGetLastError());
}

// counts (cand, nbr: device [c1 - c0]) and, with idx, the CSR fill
static hegrid_status hpx_pairs(const hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* d_cand,
                               int64_t* d_cnt, const int64_t* d_off, int64_t* d_idx, cudaStream_t st) {
    const int64_t nc = c1 - c0;
    if (nc <= 0) return HEGRID_OK;
    for (int64_t b = 0; b < nc; b += 1 << 30) {
        const int64_t m = std::min<int64_t>(nc - b, 1 << 30);
        k_hpx_pairs<<<(unsigned)m, HPX_THREADS, 0, st>>>(hpx_geom(p), p->d_keys, (uint32_t)p->n_used,
                                                        p->d_ll, p->d_perm, c0 + b,
                                                        d_cand ? d_cand + b : nullptr,
                                                        d_cnt ? d_cnt + b : nullptr,
                                                        d_off ? d_off + b : nullptr, d_idx);
        count_launch();
    }
    return cuda_status(cudaGetLastError());
}

hegrid_status hpx_neighbours(const hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* offsets,
                             int64_t* idx, cudaStream_t st) {
    const int64_t nc = c1 - c0;
    offsets[0] = 0;
    if (nc == 0) return HEGRID_OK;
    int64_t *d_cnt = nullptr, *d_off = nullptr, *d_idx = nullptr;
    std::vector<int64_t> h(nc);
    HG_TRY(plan_alloc(p, &d_cnt, nc * sizeof(int64_t), st));
    hegrid_status s = hpx_pairs(p, c0, c1, nullptr, d_cnt, nullptr, nullptr, st);
    if (s == HEGRID_OK) s = cuda_status(cudaMemcpyAsync(h.data(), d_cnt, nc * 8, cudaMemcpyDeviceToHost, st));
    if (s == HEGRID_OK) s = cuda_status(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < nc && s == HEGRID_OK; ++q) offsets[q + 1] = offsets[q] + h[q];
    const int64_t tot = offsets[nc];
    if (s == HEGRID_OK && idx && tot > 0) {
        s = cuda_status(plan_alloc(p, &d_off, nc * sizeof(int64_t), st));
        if (s == HEGRID_OK) s = cuda_status(plan_alloc(p, &d_idx, tot * sizeof(int64_t), st));
        if (s == HEGRID_OK) s = cuda_status(cudaMemcpyAsync(d_off, offsets, nc * 8, cudaMemcpyHostToDevice, st));
        if (s == HEGRID_OK) s = hpx_pairs(p, c0, c1, nullptr, nullptr, d_off, d_idx, st);
        if (s == HEGRID_OK) s = cuda_status(cudaMemcpyAsync(idx, d_idx, tot * 8, cudaMemcpyDeviceToHost, st));
        if (s == HEGRID_OK) s = cuda_status(cudaStreamSynchronize(st));
        if (s == HEGRID_OK)
            for (int64_t q = 0; q < nc; ++q) std::sort(idx + offsets[q], idx + offsets[q + 1]);
    }
    if (d_cnt) cudaFreeAsync(d_cnt, st);
    if (d_off) cudaFreeAsync(d_off, st);
    if (d_idx) cudaFreeAsync(d_idx, st);
    cudaStreamSynchronize(st);
    return s;
}

// plan statistics: candidates (the LUT's ranges) and neighbours per cell
hegrid_status hpx_pair_stats(hegrid_plan_s* p, cudaStream_t st) {
    const int64_t cells = (int64_t)p->map.nx * p->map.ny;
    hegrid_plan_stats& S = p->stats;
    S = hegrid_plan_stats{};
    if (cells == 0) return HEGRID_OK;
    int64_t *d_cand = nullptr, *d_cnt = nullptr;
    HG_TRY(plan_alloc(p, &d_cand, cells * sizeof(int64_t), st));
    HG_TRY(plan_alloc(p, &d_cnt, cells * sizeof(int64_t), st));
    hegrid_status s = hpx_pairs(p, 0, cells, d_cand, d_cnt, nullptr, nullptr, st);
    std::vector<int64_t> hc(cells), hn(cells);
    if (s == HEGRID_OK) s = cuda_status(cudaMemcpyAsync(hc.data(), d_cand, cells * 8, cudaMemcpyDeviceToHost, st));
    if (s == HEGRID_OK) s = cuda_status(cudaMemcpyAsync(hn.data(), d_cnt, cells * 8, cudaMemcpyDeviceToHost, st));
    if (s == HEGRID_OK) s = cuda_status(cudaStreamSynchronize(st));
    cudaFreeAsync(d_cand, st);
    cudaFreeAsync(d_cnt, st);
    if (s != HEGRID_OK) return s;
    int64_t mn = INT64_MAX, mx = 0, sc = 0, sn = 0;
    for (int64_t q = 0; q < cells; ++q) {
        sc += hc[q];
        sn += hn[q];
        mn = std::min(mn, hn[q]);
        mx = std::max(mx, hn[q]);
    }
    S.n_candidate_pairs = sc;
    S.n_pairs = sn;
    S.nbr_min = (int32_t)mn;
    S.nbr_max = (int32_t)mx;
    S.nbr_mean = (double)sn / cells;
    return HEGRID_OK;
}

__global__ void k_hpx_ang2pix(int64_t nside, const double* __restrict__ th, const double* __restrict__ ph,
                              int64_t n, int64_t* __restrict__ pix, int* __restrict__ bad) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double t = th[k];
    if (!isfinite(t) || !isfinite(ph[k]) || t < 0.0 || t > M_PI) {
        atomicExch(bad, 1);
        pix[k] = -1;
        return;
    }
    pix[k] = hpx::ang2pix_ring(nside, t, ph[k]);
}

}  // namespace hg

using namespace hg;

extern "C" hegrid_status hegrid_healpix_ang2pix(int32_t nside, const double* theta, const double* phi,
                                                int64_t n, int64_t* pix, int32_t device) {
    if (nside < 1 || nside > 8192 || (nside & (nside - 1)) || n < 0) return HEGRID_EINVAL;
    if (n > 0 && (!theta || !phi || !pix)) return HEGRID_EINVAL;
    if (n == 0) return HEGRID_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_status(e);
    double *dt = nullptr, *dp = nullptr;
    int64_t* dx = nullptr;
    int* db = nullptr;
    int bad = 0;
    e = cudaMalloc(&dt, n * 8);
    if (e == cudaSuccess) e = cudaMalloc(&dp, n * 8);
    if (e == cudaSuccess) e = cudaMalloc(&dx, n * 8);
    if (e == cudaSuccess) e = cudaMalloc(&db, sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(dt, theta, n * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dp, phi, n * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(db, 0, sizeof(int));
    if (e == cudaSuccess) {
        k_hpx_ang2pix<<<(unsigned)((n + 255) / 256), 256>>>(nside, dt, dp, n, dx, db);
        count_launch();
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(pix, dx, n * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&bad, db, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(dt);
    cudaFree(dp);
    cudaFree(dx);
    cudaFree(db);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_status(e);
    return bad ? HEGRID_EDOMAIN : HEGRID_OK;
}
