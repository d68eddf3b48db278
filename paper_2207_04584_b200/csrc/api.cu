// api.cu -- the C ABI (include/hegrid.h): validation, plan lifetime, the device-resident
// grid call, and the host end-to-end pipeline (channel blocks over CUDA streams with
// pinned staging; PAPER.md:279-294 multi-pipeline concurrency, :313-318 memory pool,
// pinned memory and asynchronous transfer).
#include <math.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace hg {
std::atomic<int64_t> g_launches{0};

struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    const size_t chunk = 64ull << 20;
    int nt = (int)std::min<size_t>(std::max<size_t>(bytes / chunk, 1), 16);
    if (nt <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    size_t per = (bytes + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        size_t b = t * per, e = std::min(bytes, b + per);
        if (b >= e) break;
        th.emplace_back([=] { memcpy((char*)dst + b, (const char*)src + b, e - b); });
    }
    for (auto& x : th) x.join();
}

static hegrid_status validate_geometry(const hegrid_map* m, const hegrid_kernel* k) {
    if (!m || !k) return HEGRID_EINVAL;
    if (m->nx < 1 || m->ny < 1) return HEGRID_EINVAL;
    if ((int64_t)m->nx * m->ny > (1LL << 31)) return HEGRID_EINVAL;
    const double v[] = {m->crval_lon, m->crval_lat, m->crpix_x, m->crpix_y, m->cdelt_lon,
                        m->cdelt_lat, k->fwhm_deg, k->support_sigma};
    for (double x : v)
        if (!isfinite(x)) return HEGRID_EINVAL;
    if (m->cdelt_lon == 0.0 || m->cdelt_lat == 0.0) return HEGRID_EINVAL;
    if (m->projection < HEGRID_PROJ_CAR || m->projection > HEGRID_PROJ_SIN || m->reserved != 0)
        return HEGRID_EINVAL;
    if (!(k->fwhm_deg > 0.0) || !(k->support_sigma > 0.0)) return HEGRID_EINVAL;
    if (k->kind != HEGRID_KERNEL_GAUSSIAN && k->kind != HEGRID_KERNEL_TOPHAT) return HEGRID_EINVAL;
    if (k->reserved != 0) return HEGRID_EINVAL;
    if (fabs(m->crval_lat) > 90.0) return HEGRID_EINVAL;
    return HEGRID_OK;
}

static hegrid_opts default_opts(const hegrid_opts* o) {
    hegrid_opts r{};
    if (o) r = *o;
    if (r.index < HEGRID_INDEX_AUTO || r.index > HEGRID_INDEX_HEALPIX) r.index = -1;   // rejected below
    if (r.n_streams <= 0) r.n_streams = 2;
    if (r.n_streams > 8) r.n_streams = 8;
    if (r.channel_block < 0) r.channel_block = 0;
    return r;
}

static hegrid_status create_common(const double* d_lon, const double* d_lat, int64_t n,
                                   const hegrid_map* map, const hegrid_kernel* kernel,
                                   const hegrid_opts& o, cudaStream_t st, hegrid_plan_t* out) {
    auto* p = new (std::nothrow) hegrid_plan_s();
    if (!p) return HEGRID_ENOMEM;
    p->device = o.device;
    p->map = *map;
    p->kern = *kernel;
    p->opts = o;
    p->n = n;
    {   // the device's stream-ordered pool (common.cuh): memory stays cached between calls
        // and between plans, so a new plan over the same shapes allocates nothing new
        cudaError_t e = shared_pool(o.device, &p->pool);
        if (e != cudaSuccess) {
            delete p;
            return cuda_status(e);
        }
    }
    // the spatial index: lon/lat bins where they serve the field, else (AUTO) or on request
    // the HEALPix ring-scheme LUT (hpx.cu)
    hegrid_status s = HEGRID_EUNSUPPORTED;
    if (o.index != HEGRID_INDEX_HEALPIX) s = build_plan(p, d_lon, d_lat, st);
    if ((s == HEGRID_EUNSUPPORTED && o.index == HEGRID_INDEX_AUTO) || o.index == HEGRID_INDEX_HEALPIX) {
        p->index = HEGRID_INDEX_HEALPIX;
        s = build_plan_hpx(p, d_lon, d_lat, st);
    }
    if (s != HEGRID_OK) {
        hegrid_plan_destroy(p);
        return s;
    }
    *out = p;
    return HEGRID_OK;
}

void phase_mark(const char* what) {
    static const bool on = getenv("HEGRID_TIMING") != nullptr;
    static auto t0 = std::chrono::steady_clock::now();
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    // with the device pool's reserved / used bytes (growing the pool maps new memory)
    uint64_t res = 0, used = 0;
    int dev = 0;
    cudaMemPool_t pool = nullptr;
    if (cudaGetDevice(&dev) == cudaSuccess && shared_pool(dev, &pool) == cudaSuccess) {
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    }
    fprintf(stderr, "[hegrid] %-32s %9.2f ms  pool %.2f / %.2f GB\n", what,
            std::chrono::duration<double, std::milli>(t - t0).count(), used / 1e9, res / 1e9);
    t0 = t;
}

cudaError_t shared_pool(int device, cudaMemPool_t* pool) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lock(mu);
    if (device < 0) return cudaErrorInvalidDevice;
    if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
    if (!pools[device]) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = device;
        cudaMemPool_t q = nullptr;
        cudaError_t e = cudaMemPoolCreate(&q, &pp);
        uint64_t keep = UINT64_MAX;
        if (e == cudaSuccess) e = cudaMemPoolSetAttribute(q, cudaMemPoolAttrReleaseThreshold, &keep);
        if (e != cudaSuccess) {
            if (q) cudaMemPoolDestroy(q);
            return e;
        }
        pools[device] = q;
    }
    *pool = pools[device];
    return cudaSuccess;
}

hegrid_status prepare_engine(const hegrid_plan_s* p, int64_t n_channels_per_launch) {
    if (p->index == HEGRID_INDEX_HEALPIX || p->opts.engine == HEGRID_ENGINE_SIMT || p->n_used == 0)
        return HEGRID_OK;
    auto* q = const_cast<hegrid_plan_s*>(p);
    if (!q->prep_st) HG_TRY(cudaStreamCreateWithFlags(&q->prep_st, cudaStreamNonBlocking));
    return prepare_tc(p, n_channels_per_launch, q->prep_st);
}

hegrid_status launch_accumulate(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                int64_t n_channels, float* d_out, float* d_weight,
                                cudaStream_t st) {
    // HEALPix-indexed plans have their own gather (Algorithm 1, hpx.cu).  Otherwise AUTO
    // takes the tensor-core engine: faster on every measured configuration (DESIGN.md
    // section 11: cfg2 1.5 vs 4.4 ms, cfg3 7.3 vs 109 ms, cfg4 14 vs 68 ms)
    if (p->index == HEGRID_INDEX_HEALPIX)
        return launch_accumulate_hpx(p, d_v, ldv, n_channels, d_out, d_weight, st);
    if (p->opts.engine == HEGRID_ENGINE_SIMT)
        return launch_accumulate_simt(p, d_v, ldv, n_channels, d_out, d_weight, st);
    return launch_accumulate_tc(p, d_v, ldv, n_channels, d_out, d_weight, st);
}

}  // namespace hg

using namespace hg;

extern "C" {

const char* hegrid_status_string(hegrid_status s) {
    switch (s) {
        case HEGRID_OK: return "ok";
        case HEGRID_EINVAL: return "invalid argument";
        case HEGRID_EDOMAIN: return "sample coordinate out of domain (non-finite or |lat| > 90)";
        case HEGRID_ENOMEM: return "out of memory";
        case HEGRID_ECUDA: return "CUDA error or no usable device";
        case HEGRID_EUNSUPPORTED: return "geometry not supported by the lon/lat bin index";
        case HEGRID_EINTERNAL: return "internal error";
    }
    return "unknown status";
}

int32_t hegrid_abi_version(void) { return HEGRID_ABI_VERSION; }

int64_t hegrid_launch_count(void) { return g_launches.load(); }

hegrid_status hegrid_plan_create(const double* lon_deg, const double* lat_deg, int64_t n,
                                 const hegrid_map* map, const hegrid_kernel* kernel,
                                 const hegrid_opts* opts, hegrid_plan_t* out) {
    if (!out || n < 0 || n >= (1LL << 31) - 1) return HEGRID_EINVAL;
    if (n > 0 && (!lon_deg || !lat_deg)) return HEGRID_EINVAL;
    HG_TRY_S(validate_geometry(map, kernel));
    hegrid_opts o = default_opts(opts);
    if (o.index < 0 || (o.nonfinite != HEGRID_NONFINITE_PROPAGATE && o.nonfinite != HEGRID_NONFINITE_MASK))
        return HEGRID_EINVAL;
    DeviceGuard dg(o.device);
    HG_TRY(dg.err);
    // coordinates H2D into stream-ordered buffers of the device pool (no cudaMalloc / cudaFree
    // and their device-wide synchronisation on the plan path)
    phase_mark("plan_create: enter");
    cudaMemPool_t pool = nullptr;
    HG_TRY(shared_pool(o.device, &pool));
    phase_mark("plan_create: pool");
    cudaStream_t st = nullptr;
    HG_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *d_lon = nullptr, *d_lat = nullptr;
    size_t bytes = (size_t)std::max<int64_t>(n, 1) * sizeof(double);
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&d_lon), bytes, pool, st);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&d_lat), bytes, pool, st);
    if (e == cudaSuccess && n > 0) e = cudaMemcpyAsync(d_lon, lon_deg, n * 8, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && n > 0) e = cudaMemcpyAsync(d_lat, lat_deg, n * 8, cudaMemcpyHostToDevice, st);
    hegrid_status s = cuda_status(e);
    phase_mark("plan_create: coords H2D");
    if (s == HEGRID_OK) s = create_common(d_lon, d_lat, n, map, kernel, o, st, out);
    phase_mark("plan_create: build");
    if (d_lon) cudaFreeAsync(d_lon, st);
    if (d_lat) cudaFreeAsync(d_lat, st);
    cudaError_t e2 = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    phase_mark("plan_create: done");
    if (s == HEGRID_OK && e2 != cudaSuccess) {
        hegrid_plan_destroy(*out);
        *out = nullptr;
        s = cuda_status(e2);
    }
    return s;
}

hegrid_status hegrid_plan_create_device(const double* d_lon, const double* d_lat, int64_t n,
                                        const hegrid_map* map, const hegrid_kernel* kernel,
                                        const hegrid_opts* opts, void* stream,
                                        hegrid_plan_t* out) {
    if (!out || n < 0 || n >= (1LL << 31) - 1) return HEGRID_EINVAL;
    if (n > 0 && (!d_lon || !d_lat)) return HEGRID_EINVAL;
    HG_TRY_S(validate_geometry(map, kernel));
    hegrid_opts o = default_opts(opts);
    if (o.index < 0 || (o.nonfinite != HEGRID_NONFINITE_PROPAGATE && o.nonfinite != HEGRID_NONFINITE_MASK))
        return HEGRID_EINVAL;
    DeviceGuard dg(o.device);
    HG_TRY(dg.err);
    return create_common(d_lon, d_lat, n, map, kernel, o, (cudaStream_t)stream, out);
}

void hegrid_plan_destroy(hegrid_plan_t p) {
    if (!p) return;
    DeviceGuard dg(p->device);
    phase_mark("plan_destroy: enter");
    // the plan's arrays go back to the device pool once all work issued so far is done
    cudaDeviceSynchronize();
    for (void* q : {(void*)p->d_keys, (void*)p->d_perm, (void*)p->d_iperm, (void*)p->d_geo,
                    (void*)p->d_ll, (void*)p->d_bin_start, (void*)p->d_mrow, (void*)p->d_cos_row,
                    (void*)p->d_tc_sched, (void*)p->d_tc_tile_off, (void*)p->d_tc_wsum,
                    (void*)p->d_tc_wimg, (void*)p->d_tc_wslot, (void*)p->d_omega})
        if (q) cudaFreeAsync(q, 0);
    for (auto e : p->prof_events) cudaEventDestroy(e);
    for (auto& x : p->slots) {
        if (x.st) cudaStreamSynchronize(x.st);
        for (auto e : x.ev)
            if (e) cudaEventDestroy(e);
        if (x.h_in) cudaFreeHost(x.h_in);
        if (x.h_out) cudaFreeHost(x.h_out);
        if (x.st) cudaStreamDestroy(x.st);
    }
    if (p->prep_st) cudaStreamDestroy(p->prep_st);
    cudaStreamSynchronize(0);
    delete p;
    phase_mark("plan_destroy: done");
}

__global__ void k_gather_omega(const float* __restrict__ w, const int32_t* __restrict__ perm,
                               int64_t n_used, float* __restrict__ dst) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n_used) dst[q] = w[perm[q]];
}

hegrid_status hegrid_plan_set_sample_weights(hegrid_plan_t p, const float* omega, int64_t n) {
    if (!p || (omega && n != p->n)) return HEGRID_EINVAL;
    if (omega)
        for (int64_t k = 0; k < n; ++k)
            if (!(omega[k] >= 0.0f) || !isfinite(omega[k])) return HEGRID_EDOMAIN;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    HG_TRY(cudaDeviceSynchronize());
    // the engine tables that hold weights (W per cell, the weight image) are rebuilt lazily;
    // the tensor-core schedule is geometric but is rebuilt with them
    for (void* q : {(void*)p->d_tc_sched, (void*)p->d_tc_tile_off, (void*)p->d_tc_wsum,
                    (void*)p->d_tc_wimg, (void*)p->d_tc_wslot})
        if (q) cudaFreeAsync(q, 0);
    p->d_tc_sched = nullptr;
    p->d_tc_tile_off = nullptr;
    p->d_tc_wsum = nullptr;
    p->d_tc_wimg = nullptr;
    p->d_tc_wslot = nullptr;
    p->tc_nchunks = -1;
    p->tc_pw = -1;
    p->tc_wimg_bytes = 0;
    if (p->d_omega) cudaFreeAsync(p->d_omega, 0);
    p->d_omega = nullptr;
    if (!omega || p->n_used == 0) return cuda_status(cudaStreamSynchronize(0));
    float* d_w = nullptr;
    HG_TRY(plan_alloc(p, &d_w, n * sizeof(float), 0));
    cudaError_t e = plan_alloc(p, &p->d_omega, p->n_used * sizeof(float), 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_w, omega, n * sizeof(float), cudaMemcpyHostToDevice, 0);
    if (e == cudaSuccess) {
        k_gather_omega<<<(unsigned)((p->n_used + 255) / 256), 256, 0, 0>>>(d_w, p->d_perm, p->n_used, p->d_omega);
        count_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(d_w, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    if (e != cudaSuccess && p->d_omega) {
        cudaFreeAsync(p->d_omega, 0);
        p->d_omega = nullptr;
    }
    return cuda_status(e);
}

hegrid_status hegrid_plan_info(hegrid_plan_t p, hegrid_plan_stats* out) {
    if (!p || !out) return HEGRID_EINVAL;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    if (!p->stats_valid) {
        if (p->index == HEGRID_INDEX_HEALPIX) HG_TRY_S(hpx_pair_stats(p, 0));
        else HG_TRY_S(plan_pair_stats(p, 0));
        p->stats_valid = true;
    }
    hegrid_plan_stats s = p->stats;
    s.n_samples = p->n;
    s.n_used = p->n_used;
    s.n_bins = p->g.nbins;
    s.t_plan_ms = p->t_plan_ms;
    s.nrow = p->g.nrow;
    s.ncol = p->g.ncol;
    s.mlat = p->g.mlat;
    s.mlon = p->g.mlon;
    s.sigma_deg = p->g.sigma_rad / kDeg2Rad;
    s.radius_deg = p->g.R_rad / kDeg2Rad;
    s.weight_image_bytes = p->tc_pw == 1 ? p->tc_wimg_bytes : 0;
    s.index = p->index;
    s.nside = p->hpx_nside;
    s.tc_entries = p->tc_nchunks > 0 ? p->tc_nchunks : 0;
    s.tc_block_slots = p->tc_nchunks > 0 ? (int64_t)p->tc_stats[1] : 0;
    *out = s;
    return HEGRID_OK;
}

hegrid_status hegrid_plan_permutation(hegrid_plan_t p, int64_t* perm, int64_t* n_used) {
    if (!p) return HEGRID_EINVAL;
    if (n_used) *n_used = p->n_used;
    if (!perm || p->n_used == 0) return HEGRID_OK;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    std::vector<int32_t> h(p->n_used);
    HG_TRY(cudaMemcpy(h.data(), p->d_perm, p->n_used * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < p->n_used; ++i) perm[i] = h[i];
    return HEGRID_OK;
}

hegrid_status hegrid_permute_device(hegrid_plan_t p, const float* d_user, int64_t n_channels,
                                    int64_t ld_user, float* d_plan, int64_t ld_plan,
                                    void* stream) {
    if (!p || n_channels < 0) return HEGRID_EINVAL;
    if (n_channels == 0) return HEGRID_OK;
    if (!d_user || !d_plan || ld_user < p->n || ld_plan < n_channels || ld_plan % 4) return HEGRID_EINVAL;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    return launch_permute(p, d_user, n_channels, ld_user, d_plan, ld_plan, (cudaStream_t)stream);
}

static hegrid_status accumulate_profiled(hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                         int64_t C, float* d_out, float* d_w, cudaStream_t st) {
    if (!p->profile) return launch_accumulate(p, d_v, ldv, C, d_out, d_w, st);
    cudaEvent_t a, b;
    HG_TRY(cudaEventCreate(&a));
    HG_TRY(cudaEventCreate(&b));
    HG_TRY(cudaEventRecord(a, st));
    hegrid_status s = launch_accumulate(p, d_v, ldv, C, d_out, d_w, st);
    HG_TRY(cudaEventRecord(b, st));
    p->prof_events.push_back(a);
    p->prof_events.push_back(b);
    return s;
}

// W only (n_channels == 0 but a weight map was requested): one pass over a zero row.
static hegrid_status weights_only(hegrid_plan_s* p, float* d_w, cudaStream_t st) {
    float* z = nullptr;
    float* o = nullptr;
    size_t nz = (size_t)std::max<int64_t>(p->n_used, 1) * 4;
    HG_TRY(plan_alloc(p, &z, nz * sizeof(float), st));
    HG_TRY(plan_alloc(p, &o, (size_t)p->g.nx * p->g.ny * sizeof(float), st));
    HG_TRY(cudaMemsetAsync(z, 0, nz * sizeof(float), st));
    hegrid_status s = launch_accumulate(p, z, 4, 1, o, d_w, st);
    cudaFreeAsync(z, st);
    cudaFreeAsync(o, st);
    return s;
}

hegrid_status hegrid_grid_device(hegrid_plan_t p, const float* d_data, int64_t n_channels,
                                 int64_t ld, int32_t layout, float* d_out, float* d_weight,
                                 void* stream) {
    if (!p || n_channels < 0) return HEGRID_EINVAL;
    if (n_channels > 0 && (!d_data || !d_out)) return HEGRID_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    if (n_channels == 0) return d_weight ? weights_only(p, d_weight, st) : HEGRID_OK;
    const int64_t cells = (int64_t)p->g.nx * p->g.ny;
    if (layout == HEGRID_LAYOUT_PLAN_NC) {
        if (ld < n_channels || ld % 4 || ((uintptr_t)d_data & 15)) return HEGRID_EINVAL;
        return accumulate_profiled(p, d_data, ld, n_channels, d_out, d_weight, st);
    }
    if (layout != HEGRID_LAYOUT_USER_CN) return HEGRID_EINVAL;
    if (ld < p->n) return HEGRID_EINVAL;
    // USER_CN: permute channel blocks through a plan-layout scratch, stream-ordered from the
    // plan's pool on the caller's stream (no buffer shared between streams)
    int64_t cb = std::min<int64_t>(n_channels, 512);
    cb = (cb + 3) & ~3LL;
    size_t need = (size_t)std::max<int64_t>(p->n_used, 1) * cb * sizeof(float);
    float* scratch = nullptr;
    HG_TRY(plan_alloc(p, &scratch, need, st));
    hegrid_status s = HEGRID_OK;
    for (int64_t c0 = 0; c0 < n_channels && s == HEGRID_OK; c0 += cb) {
        int64_t cn = std::min(cb, n_channels - c0);
        s = launch_permute(p, d_data + c0 * ld, cn, ld, scratch, cb, st);
        if (s == HEGRID_OK)
            s = accumulate_profiled(p, scratch, cb, cn, d_out + c0 * cells,
                                    c0 == 0 ? d_weight : nullptr, st);
    }
    cudaError_t e = cudaFreeAsync(scratch, st);
    if (s == HEGRID_OK) s = cuda_status(e);
    return s;
}

hegrid_status hegrid_grid(hegrid_plan_t p, const float* data, int64_t n_channels,
                          float* out_map, float* weight_map) {
    if (!p || n_channels < 0) return HEGRID_EINVAL;
    if (n_channels > 0 && (!out_map || (p->n > 0 && !data))) return HEGRID_EINVAL;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    const int64_t cells = (int64_t)p->g.nx * p->g.ny;
    const int64_t n = p->n;
    if (n_channels == 0) {
        if (!weight_map) return HEGRID_OK;
        float* d_w = nullptr;
        HG_TRY(plan_alloc(p, &d_w, cells * sizeof(float), 0));
        hegrid_status s = weights_only(p, d_w, 0);
        if (s == HEGRID_OK) s = cuda_status(cudaMemcpy(weight_map, d_w, cells * 4, cudaMemcpyDeviceToHost));
        cudaFreeAsync(d_w, 0);
        cudaStreamSynchronize(0);
        return s;
    }
    int64_t cb = p->opts.channel_block > 0 ? p->opts.channel_block
                                           : (n_channels >= 1024 ? 512 : 256);
    cb = std::min<int64_t>(cb, n_channels);
    cb = (cb + 3) & ~3LL;
    const int S = p->opts.n_streams;
    const int64_t nblk = (n_channels + cb - 1) / cb;
    const bool in_pinned = n == 0 || is_pinned(data);
    const bool out_pinned = is_pinned(out_map);
    const size_t raw_b = (size_t)cb * std::max<int64_t>(n, 1) * 4;
    const size_t v_b = (size_t)cb * std::max<int64_t>(p->n_used, 1) * 4;
    const size_t out_b = (size_t)cb * cells * 4;
    hegrid_status s = HEGRID_OK;
    auto fail = [&](cudaError_t e) {
        if (s == HEGRID_OK && e != cudaSuccess) s = cuda_status(e);
        return s != HEGRID_OK;
    };
    // the plan's staging slots (streams, events, pinned buffers) persist across calls
    while ((int)p->slots.size() < S && s == HEGRID_OK) {
        hegrid_plan_s::StageSlot x;
        if (fail(cudaStreamCreateWithFlags(&x.st, cudaStreamNonBlocking))) break;
        for (auto& e : x.ev)
            if (fail(cudaEventCreate(&e))) break;
        p->slots.push_back(x);
    }
    auto grow = [&](float** h, size_t* cap, size_t need) {
        if (*cap >= need) return;
        if (*h) cudaFreeHost(*h);
        *h = nullptr;
        *cap = 0;
        if (!fail(cudaHostAlloc(h, need, cudaHostAllocDefault))) *cap = need;
    };
    struct Dev {
        float *raw = nullptr, *v = nullptr, *out = nullptr;
        int64_t pending = -1;   // block whose output waits in the slot's pinned buffer
    };
    std::vector<Dev> dv(S);
    for (int k = 0; k < S && s == HEGRID_OK; ++k) {
        auto& x = p->slots[k];
        if (!in_pinned) grow(&x.h_in, &x.in_cap, raw_b);
        if (!out_pinned) grow(&x.h_out, &x.out_cap, out_b);
        if (s != HEGRID_OK) break;
        if (fail(plan_alloc(p, &dv[k].raw, raw_b, x.st))) break;
        if (fail(plan_alloc(p, &dv[k].v, v_b, x.st))) break;
        if (fail(plan_alloc(p, &dv[k].out, out_b, x.st))) break;
    }
    float* d_w = nullptr;
    if (s == HEGRID_OK && weight_map) fail(plan_alloc(p, &d_w, cells * sizeof(float), p->slots[0].st));
    // pipeline trace (profiling): four timing events per block on its slot's stream
    const bool trace = p->profile;
    std::vector<cudaEvent_t> tev;
    if (trace && s == HEGRID_OK) {
        tev.assign(4 * nblk, nullptr);
        for (auto& e : tev)
            if (fail(cudaEventCreate(&e))) break;
    }
    auto mark = [&](int64_t b, int k, cudaStream_t st) {
        if (trace) fail(cudaEventRecord(tev[4 * b + k], st));
    };
    auto drain = [&](int k) {
        Dev& d = dv[k];
        if (d.pending < 0) return;
        if (fail(cudaEventSynchronize(p->slots[k].ev[3]))) return;
        if (!out_pinned) {
            int64_t c0 = d.pending * cb, cn = std::min(cb, n_channels - c0);
            parallel_memcpy(out_map + c0 * cells, p->slots[k].h_out, (size_t)cn * cells * 4);
        }
        d.pending = -1;
    };
    for (int64_t b = 0; b < nblk && s == HEGRID_OK; ++b) {
        const int k = (int)(b % S);
        auto& x = p->slots[k];
        Dev& d = dv[k];
        drain(k);
        if (s != HEGRID_OK) break;
        const int64_t c0 = b * cb, cn = std::min(cb, n_channels - c0);
        mark(b, 0, x.st);
        if (n > 0) {
            const float* src = data + c0 * n;
            if (!in_pinned) {
                parallel_memcpy(x.h_in, src, (size_t)cn * n * 4);
                src = x.h_in;
            }
            if (fail(cudaMemcpyAsync(d.raw, src, (size_t)cn * n * 4, cudaMemcpyHostToDevice, x.st)))
                break;
            mark(b, 1, x.st);
            // the engine's one-time per-plan tables (tensor-core schedule, W, weight image) are
            // built on the plan's own stream while the first block is in flight over PCIe
            if (b == 0 && (s = prepare_engine(p, std::min(cb, n_channels))) != HEGRID_OK) break;
            if ((s = launch_permute(p, d.raw, cn, n, d.v, cb, x.st)) != HEGRID_OK) break;
        } else {
            mark(b, 1, x.st);
        }
        if ((s = launch_accumulate(p, d.v, cb, cn, d.out, b == 0 ? d_w : nullptr, x.st)) != HEGRID_OK)
            break;
        mark(b, 2, x.st);
        float* dst = out_pinned ? out_map + c0 * cells : x.h_out;
        if (fail(cudaMemcpyAsync(dst, d.out, (size_t)cn * cells * 4, cudaMemcpyDeviceToHost, x.st)))
            break;
        mark(b, 3, x.st);
        if (fail(cudaEventRecord(x.ev[3], x.st))) break;
        d.pending = b;
    }
    for (int k = 0; k < S; ++k) drain(k);
    if (s == HEGRID_OK && weight_map) {
        fail(cudaStreamSynchronize(p->slots[0].st));
        if (s == HEGRID_OK) fail(cudaMemcpy(weight_map, d_w, cells * 4, cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < S && k < (int)p->slots.size(); ++k) {
        cudaStream_t st = p->slots[k].st;
        if (dv[k].raw) cudaFreeAsync(dv[k].raw, st);
        if (dv[k].v) cudaFreeAsync(dv[k].v, st);
        if (dv[k].out) cudaFreeAsync(dv[k].out, st);
        if (k == 0 && d_w) cudaFreeAsync(d_w, st);
        cudaStreamSynchronize(st);
    }
    if (trace) {
        p->trace.clear();
        if (s == HEGRID_OK) {
            for (int64_t b = 0; b < nblk; ++b) {
                p->trace.push_back((double)(b % S));
                for (int k = 0; k < 4; ++k) {
                    float ms = 0;
                    fail(cudaEventElapsedTime(&ms, tev[0], tev[4 * b + k]));
                    p->trace.push_back(ms);
                }
            }
        }
        for (auto e : tev)
            if (e) cudaEventDestroy(e);
    }
    return s;
}

hegrid_status hegrid_neighbours(hegrid_plan_t p, int64_t cell_begin, int64_t cell_end,
                                int64_t* offsets, int64_t* sample_idx) {
    if (!p || !offsets) return HEGRID_EINVAL;
    int64_t cells = (int64_t)p->g.nx * p->g.ny;
    if (cell_begin < 0 || cell_end < cell_begin || cell_end > cells) return HEGRID_EINVAL;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    // the pairs of the engine that grids: the HEALPix gather's ring ranges, the tensor-core
    // engine's chunk schedule (the default), or the SIMT engine's per-cell candidate ranges
    if (p->index == HEGRID_INDEX_HEALPIX)
        return hpx_neighbours(p, cell_begin, cell_end, offsets, sample_idx, 0);
    if (p->opts.engine == HEGRID_ENGINE_SIMT)
        return plan_neighbours(p, cell_begin, cell_end, offsets, sample_idx, 0);
    return tc_neighbours(p, cell_begin, cell_end, offsets, sample_idx, 0);
}

hegrid_status hegrid_sort_u32(const uint32_t* keys, int64_t n, int32_t* perm, int32_t device) {
    if (n < 0 || n >= (1LL << 31) - 1 || (n > 0 && (!keys || !perm))) return HEGRID_EINVAL;
    if (n == 0) return HEGRID_OK;
    DeviceGuard dg(device);
    HG_TRY(dg.err);
    uint32_t* dk = nullptr;
    int32_t* dv = nullptr;
    std::vector<int32_t> iota(n);
    for (int64_t i = 0; i < n; ++i) iota[i] = (int32_t)i;
    HG_TRY(cudaMalloc(&dk, n * 4));
    cudaError_t e = cudaMalloc(&dv, n * 4);
    if (e == cudaSuccess) e = cudaMemcpy(dk, keys, n * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dv, iota.data(), n * 4, cudaMemcpyHostToDevice);
    hegrid_status s = cuda_status(e);
    if (s == HEGRID_OK) s = radix_sort_pairs(dk, dv, n, 32, 0);
    if (s == HEGRID_OK) s = cuda_status(cudaMemcpy(perm, dv, n * 4, cudaMemcpyDeviceToHost));
    cudaFree(dk);
    if (dv) cudaFree(dv);
    return s;
}

hegrid_status hegrid_pipeline_trace(hegrid_plan_t p, double* buf, int64_t cap_rows,
                                    int64_t* n_rows) {
    if (!p || cap_rows < 0) return HEGRID_EINVAL;
    const int64_t rows = (int64_t)p->trace.size() / 5;
    if (n_rows) *n_rows = rows;
    if (buf)
        for (int64_t i = 0; i < std::min(rows, cap_rows) * 5; ++i) buf[i] = p->trace[i];
    return HEGRID_OK;
}

hegrid_status hegrid_profile_enable(hegrid_plan_t p, int32_t enable) {
    if (!p) return HEGRID_EINVAL;
    p->profile = enable != 0;
    return HEGRID_OK;
}

hegrid_status hegrid_profile_read(hegrid_plan_t p, double* ms, int64_t* launches) {
    if (!p) return HEGRID_EINVAL;
    DeviceGuard dg(p->device);
    HG_TRY(dg.err);
    double tot = 0;
    int64_t k = 0;
    hegrid_status s = HEGRID_OK;
    for (size_t i = 0; i + 1 < p->prof_events.size(); i += 2) {
        float x = 0;
        cudaError_t e = cudaEventSynchronize(p->prof_events[i + 1]);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&x, p->prof_events[i], p->prof_events[i + 1]);
        if (e != cudaSuccess) s = cuda_status(e);
        tot += x;
        ++k;
    }
    for (auto e : p->prof_events) cudaEventDestroy(e);
    p->prof_events.clear();
    if (ms) *ms = tot;
    if (launches) *launches = k;
    return s;
}

}  // extern "C"
