// common.cuh -- internal types shared by the hegrid CUDA translation units.
// Nothing here is part of the ABI (include/hegrid.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <vector>

#include "../../include/hegrid.h"

namespace hg {

extern std::atomic<int64_t> g_launches;
inline void count_launch(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

constexpr double kPi = 3.14159265358979323846;
constexpr double kDeg2Rad = kPi / 180.0;
// largest half-longitude offset (rad) of a pair within R that the fp32 series distance
// serves (weight.cuh sin2_series; make_geom refuses wider reaches)
constexpr double kMaxHalfDlon = 0.5;

// Geometry of the bin index and kernel, passed by value to kernels.
// Bin (br, bc) of the index covers the cell-sized box around cell (bc - mlon, br - mlat);
// the bin grid is nrow x ncol = (ny + 2 mlat) x (nx + 2 mlon); key = br * ncol + bc,
// samples that cannot reach any cell get key = nbins (sorted to the end, never read).
struct Geom {
    int nx, ny;
    int nrow, ncol, mlat, mlon;
    int rl;                 // bin-row reach of a cell row (rows j-rl .. j+rl)
    int64_t nbins;
    // fp64 map header (cell centres, fp64 recheck)
    double crval_lon, crval_lat, crpix_x, crpix_y, cdelt_lon, cdelt_lat;
    double R_rad, sigma_rad;
    // fp32 constants of the hot-path weight
    float dlon_rad, dlat_rad;   // cdelt in radians (signed)
    float R2_lo, R2_hi;         // guard band around R^2 (rad^2): below -> in, above -> out
    float neg_k2;               // -log2(e) / (2 sigma^2)  (w = 2^(d^2 * neg_k2))
    // the same, folded into the exponent t = neg_k2 d^2 = h (K0 + h (K1 + h K2)) of the
    // tensor-core engine's weight patches; t >= t_in: inside, t < t_out: outside, else the
    // guard band (t_in = neg_k2 R2_lo, t_out = neg_k2 R2_hi; neg_k2 < 0 flips the order)
    float tK0, tK1, tK2, t_in, t_out;
    // kernel shape: w = 2^(wexp * t): wexp = 1 for the Gaussian, 0 for the tophat (w = 1
    // inside the support; the support test keeps using the Gaussian-scaled t)
    float wexp;
};

// Per-sample plan data in plan order.
// geo = { x offset from bin centre (cells), y offset (cells), cos(lat), bin column (as int bits) }
struct PlanDev {
    const float4* geo;
    const double2* ll;          // fp64 (lon, lat) deg, plan order (guard-band recheck)
    const uint32_t* bin_start;  // [nbins + 1]
    const int* mrow;            // [nrow] lon reach (bins) of a cell for samples in that bin row
    const float* cos_row;       // [ny] cos(lat) of cell rows (fp32)
    const float* omega;         // [n_used] per-sample weights in plan order (nullptr = all 1)
};

}  // namespace hg

struct hegrid_plan_s {
    int device = 0;
    int index = HEGRID_INDEX_BINS;   // the plan's spatial index (hegrid_index)
    int hpx_nside = 0;               // HEALPIX: resolution of the ring-scheme keys (hpx.cu)
    hegrid_map map{};
    hegrid_kernel kern{};
    hegrid_opts opts{};
    int64_t n = 0, n_used = 0;
    hg::Geom g{};
    // device arrays
    uint32_t* d_keys = nullptr;     // sorted keys [n]
    int32_t* d_perm = nullptr;      // plan position -> original index [n]
    int32_t* d_iperm = nullptr;     // original index -> plan position [n]
    float4* d_geo = nullptr;        // [n_used]
    double2* d_ll = nullptr;        // [n_used]
    uint32_t* d_bin_start = nullptr;
    int* d_mrow = nullptr;
    float* d_cos_row = nullptr;
    float* d_omega = nullptr;       // per-sample weights, plan order (hegrid_plan_set_sample_weights)
    double t_plan_ms = 0;
    int64_t max_cand = 0;           // max candidate-range length over cells
    bool stats_valid = false;
    hegrid_plan_stats stats{};
    // profiling
    bool profile = false;
    std::vector<cudaEvent_t> prof_events;  // start/stop pairs
    // tensor-core engine: per-tile chunk schedule (built on first use, see grid_tc.cu)
    mutable uint4* d_tc_sched = nullptr;       // {plan position, n samples, bin row, block mask}
    mutable uint32_t* d_tc_tile_off = nullptr; // [tiles + 1]
    mutable int64_t tc_nchunks = -1;
    mutable uint32_t tc_max_cpb = 0;           // max schedule entries touching one block
    mutable uint32_t tc_stats[5] = {0, 0, 0, 0, 0};  // chunks, (chunk, block) pairs, samples, runs, spans
    mutable float* d_tc_wsum = nullptr;        // [cells] W with the TC engine's weights
    // precomputed weight image (grid_tc.cu, "PW" mode): per schedule entry, its in-reach
    // blocks' tf32 hi then lo weights in the shared-memory operand layout (4 KB per block)
    mutable uint8_t* d_tc_wimg = nullptr;
    mutable uint32_t* d_tc_wslot = nullptr;    // [entries] first 4-KB slot of each entry
    mutable int tc_pw = -1;                    // -1 not built (retried on later calls), 1 built
    mutable int64_t tc_wimg_bytes = 0;
    // Stream-ordered device memory pool (the paper's per-stream "memory pool",
    // PAPER.md:315-316): every device buffer of the plan (its arrays, the engine tables and
    // weight image, and per call the USER_CN scratch, split-tile partial sums, non-finite
    // records, hegrid_grid's channel-block slots) is taken from it on the caller's stream
    // and returned to it on the same stream, so calls on different streams never share a
    // buffer and repeated calls (and later plans) reuse the memory (release threshold:
    // never).  One pool per device, shared by all plans of the process.
    cudaMemPool_t pool = nullptr;      // the device's shared pool (shared_pool), not owned
    cudaStream_t prep_st = nullptr;    // one-time engine preparation (prepare_engine)
    // hegrid_grid's staging slots, created on first use and reused by later calls: one CUDA
    // stream, its events and pinned host buffers (grown on demand) per slot
    struct StageSlot {
        cudaStream_t st = nullptr;
        cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};   // h2d start/end, compute end, d2h end
        float* h_in = nullptr;
        float* h_out = nullptr;
        size_t in_cap = 0, out_cap = 0;
    };
    std::vector<StageSlot> slots;
    // pipeline trace of the last hegrid_grid call (profiling on): per channel block
    // {slot, t_h2d_start, t_h2d_end, t_compute_end, t_d2h_end} (ms from the first event)
    std::vector<double> trace;

    hg::PlanDev dev() const {
        return hg::PlanDev{d_geo, d_ll, d_bin_start, d_mrow, d_cos_row, d_omega};
    }
};

namespace hg {

// plan.cu
hegrid_status build_plan(hegrid_plan_s* p, const double* d_lon, const double* d_lat,
                         cudaStream_t st);
hegrid_status radix_sort_pairs(uint32_t* d_keys, int32_t* d_vals, int64_t n, int bits,
                               cudaStream_t st);
hegrid_status plan_pair_stats(hegrid_plan_s* p, cudaStream_t st);
hegrid_status plan_neighbours(hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* offsets,
                              int64_t* idx, cudaStream_t st);

// hpx.cu (HEALPix-indexed plans)
hegrid_status build_plan_hpx(hegrid_plan_s* p, const double* d_lon, const double* d_lat,
                             cudaStream_t st);
hegrid_status launch_accumulate_hpx(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                    int64_t n_channels, float* d_out, float* d_weight,
                                    cudaStream_t st);
hegrid_status hpx_neighbours(const hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* offsets,
                             int64_t* idx, cudaStream_t st);
hegrid_status hpx_pair_stats(hegrid_plan_s* p, cudaStream_t st);

// grid_simt.cu
hegrid_status launch_accumulate_simt(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                     int64_t n_channels, float* d_out, float* d_weight,
                                     cudaStream_t st);
// grid_tc.cu
hegrid_status launch_accumulate_tc(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                   int64_t n_channels, float* d_out, float* d_weight,
                                   cudaStream_t st);
hegrid_status tc_neighbours(const hegrid_plan_s* p, int64_t c0, int64_t c1, int64_t* offsets,
                            int64_t* idx, cudaStream_t st);
// engine dispatch (api.cu)
hegrid_status launch_accumulate(const hegrid_plan_s* p, const float* d_v, int64_t ldv,
                                int64_t n_channels, float* d_out, float* d_weight,
                                cudaStream_t st);
// permute.cu
hegrid_status launch_permute(const hegrid_plan_s* p, const float* d_user, int64_t n_channels,
                             int64_t ld_user, float* d_plan, int64_t ld_plan, cudaStream_t st);

// api.cu: the process-wide stream-ordered pool of a device (release threshold: never)
cudaError_t shared_pool(int device, cudaMemPool_t* pool);
// grid_tc.cu / api.cu: build the engine's per-plan tables now (on the plan's prep stream)
hegrid_status prepare_engine(const hegrid_plan_s* p, int64_t n_channels_per_launch);
hegrid_status prepare_tc(const hegrid_plan_s* p, int64_t n_channels_per_launch, cudaStream_t st);

// HEGRID_TIMING=1: host-side phase timer (stderr), for the one-time plan / engine costs
void phase_mark(const char* what);

inline cudaError_t plan_alloc(const hegrid_plan_s* p, void* ptr, size_t bytes, cudaStream_t st) {
    return cudaMallocFromPoolAsync(reinterpret_cast<void**>(ptr), bytes, p->pool, st);
}

// stream-ordered scratch from the current device's pool (never trimmed, unlike the default
// pool, which returns its memory at every synchronisation)
inline cudaError_t scratch_alloc(void* ptr, size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaMemPool_t pool = nullptr;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = shared_pool(dev, &pool);
    if (e != cudaSuccess) return e;
    return cudaMallocFromPoolAsync(reinterpret_cast<void**>(ptr), bytes, pool, st);
}

inline hegrid_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return HEGRID_OK;
    if (e == cudaErrorMemoryAllocation) return HEGRID_ENOMEM;
    return HEGRID_ECUDA;
}

}  // namespace hg

#define HG_TRY(expr)                                         \
    do {                                                     \
        cudaError_t _e = (expr);                             \
        if (_e != cudaSuccess) return hg::cuda_status(_e);   \
    } while (0)

#define HG_TRY_S(expr)                      \
    do {                                    \
        hegrid_status _s = (expr);          \
        if (_s != HEGRID_OK) return _s;     \
    } while (0)
