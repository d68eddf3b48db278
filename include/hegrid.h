/*
 * hegrid.h -- C ABI of the B200-native HEGrid gridding hot path.
 *
 * The operation (Sec. 2.2, Eq. 1): N non-uniform samples s_n with
 * equatorial coordinates (alpha_n, delta_n) and C channel values V_c[s_n] are gridded
 * onto an I x J regular lon/lat map:
 *
 *     V_c[g_ij] = (1 / W_ij) * sum_n V_c[s_n] w(alpha_ij, delta_ij; alpha_n, delta_n),
 *     W_ij      = sum_n w(alpha_ij, delta_ij; alpha_n, delta_n),
 *
 * w = exp(-d^2 / 2 sigma^2) for great-circle distance d <= R, else 0 (Algorithm 1,
 * "if d(target_cell[], raw_data[i]) <= R ... Compute the weight sum,
 * Compute the weighted value ... Normalize the weighted value").  All channels share
 * the coordinates, so the spatial index ("LUT", steps 1,2,4) and
 * every (cell, sample) weight are built/computed once per plan or per launch and
 * shared by all channels (the paper's component-share redundancy elimination,
 * PAPER.md:297-305).
 *
 * Conventions (apply to every entry point):
 *   - Every call returns hegrid_status; HEGRID_OK == 0.  No exception, abort or exit
 *     crosses the ABI.  hegrid_status_string() names a code.
 *   - Angles are degrees (fp64) at the boundary.  Sample values and outputs are fp32.
 *   - Input pointers are BORROWED for the duration of the call only (for the
 *     *_device calls: until the work enqueued on `stream` completes).  Outputs are
 *     caller-allocated.  On error the contents of outputs are unspecified and the
 *     plan is unchanged.
 *   - A plan is immutable after creation, owns all of its device memory, and is bound
 *     to one CUDA device (opts->device).  Calls on one plan must be serialised by the
 *     caller.  Multi-GPU = one plan per device / process.
 *   - Host pointers may be pageable or pinned; pinned (cudaHostAlloc'd or registered)
 *     host buffers are transferred by DMA directly, pageable ones via an internal
 *     pinned staging pool.
 *   - Blank cells (W = 0) get NaN in out_map and 0 in weight_map (reading R8).
 *   - The library contains no CPU fallback: every numeric step runs in its sm_100a
 *     kernels.  Without a usable device, calls that compute return HEGRID_ECUDA.
 */
#ifndef HEGRID_H
#define HEGRID_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEGRID_ABI_VERSION 4

typedef enum hegrid_status {
    HEGRID_OK = 0,
    HEGRID_EINVAL = 1,       /* NULL pointer, n < 0, nx/ny < 1, fwhm <= 0, support <= 0,
                                cdelt == 0, bad layout/stride/alignment, n >= 2^31 */
    HEGRID_EDOMAIN = 2,      /* non-finite lon/lat or |lat| > 90 in the samples */
    HEGRID_ENOMEM = 3,       /* device or pinned host allocation failed */
    HEGRID_ECUDA = 4,        /* CUDA runtime error or no usable device */
    HEGRID_EUNSUPPORTED = 5, /* geometry outside this build's lon/lat bin index: kernel
                                radius R > 1 deg, map + R reaching a pole, or map + R
                                spanning >= 180 deg of longitude (HEALPix index: NEXT-2) */
    HEGRID_EINTERNAL = 6
} hegrid_status;

/* Regular lon/lat ("plate carree") target grid, "regular, uniform grid
 * with I x J cells"; FITS-like header (reading R6).  Cell (i, j), 0-based, i fastest:
 *     lon_ij = crval_lon + (i + 1 - crpix_x) * cdelt_lon
 *     lat_ij = crval_lat + (j + 1 - crpix_y) * cdelt_lat
 * crpix_* are 1-based reference pixels ((n + 1) / 2 centres the map on crval).
 * cdelt_* may be negative; must be non-zero. */
typedef struct hegrid_map {
    int32_t nx, ny;                 /* I (lon), J (lat) */
    double crval_lon, crval_lat;    /* deg */
    double crpix_x, crpix_y;        /* 1-based */
    double cdelt_lon, cdelt_lat;    /* deg per cell */
    int32_t projection;             /* hegrid_projection */
    int32_t reserved;               /* must be 0 */
} hegrid_map;

/* Cell centres of the map (reading R26).  Intermediate world coordinates of cell (i, j):
 * x = (i + 1 - crpix_x) cdelt_lon, y = (j + 1 - crpix_y) cdelt_lat (deg).
 * CAR: the linear lon/lat grid of the paper's "regular, uniform grid" (reading
 *      R6): lon = crval_lon + x, lat = crval_lat + y.
 * TAN / SIN: the zenithal gnomonic / orthographic projections of the FITS WCS standard
 *      (Calabretta & Greisen 2002) with the reference point (crval_lon, crval_lat) at the
 *      native pole and LONPOLE = 180 deg: the cell lies at great-circle distance atan(r)
 *      (TAN) or asin(r) (SIN) from the reference point, r = sqrt(x^2 + y^2) in radians,
 *      in the direction of position angle atan2(x, y) (NEXT-4).  Projected maps are served
 *      by the HEALPix index (the lon/lat bins need CAR). */
typedef enum hegrid_projection {
    HEGRID_PROJ_CAR = 0,
    HEGRID_PROJ_TAN = 1,
    HEGRID_PROJ_SIN = 2
} hegrid_projection;

/* Convolution kernel w(d) of the great-circle distance d (readings R1-R3; SPEC.md:117-126
 * KernelSpec{kind, sigma, radius}): sigma = fwhm / (2 sqrt(2 ln 2)), support radius
 * R = support_sigma * sigma (the paper's R).
 *   HEGRID_KERNEL_GAUSSIAN (0): w = exp(-d^2 / (2 sigma^2)) for d <= R, else 0;
 *   HEGRID_KERNEL_TOPHAT   (1): w = 1 for d <= R, else 0 (sigma only sets R).
 * Zero-initialised structs select the Gaussian.  Other kinds: HEGRID_EINVAL. */
typedef enum hegrid_kernel_kind {
    HEGRID_KERNEL_GAUSSIAN = 0,
    HEGRID_KERNEL_TOPHAT = 1
} hegrid_kernel_kind;

typedef struct hegrid_kernel {
    double fwhm_deg;        /* > 0 */
    double support_sigma;   /* > 0; 3 is the usual choice */
    int32_t kind;           /* hegrid_kernel_kind */
    int32_t reserved;       /* must be 0 */
} hegrid_kernel;

typedef enum hegrid_engine {
    HEGRID_ENGINE_AUTO = 0,   /* library picks (currently the tensor-core engine) */
    HEGRID_ENGINE_SIMT = 1,   /* FP32 SIMT accumulate (register-blocked, lanes own channels) */
    HEGRID_ENGINE_TC = 2      /* tcgen05 tensor cores, error-compensated (fp32-accurate): tf32 hi*hi + bf16 corrections */
} hegrid_engine;

/* Optional knobs; pass NULL for defaults. */
typedef struct hegrid_opts {
    int32_t device;         /* CUDA device ordinal (default 0) */
    int32_t n_streams;      /* streams for hegrid_grid's channel-block pipeline (0 = 2) */
    int32_t channel_block;  /* channels per pipeline block in hegrid_grid (0 = auto; rounded
                               up to a multiple of 4) */
    int32_t engine;         /* hegrid_engine */
    int64_t weight_image_max_bytes;  /* tensor-core engine: cap on the plan's precomputed weight
                               image (every (cell, sample) weight of the chunk schedule, built
                               once per plan on first use and kept for the plan's lifetime;
                               DESIGN.md sec. 6).  0 = auto (at most 1/4 of the device memory
                               free at build time), > 0 = at most this many bytes, < 0 = never
                               (weights computed in every launch).  A plan whose image did not
                               fit retries on later calls. */
    int32_t index;          /* hegrid_index: the plan's spatial index */
    int32_t nonfinite;      /* hegrid_nonfinite: how non-finite sample values enter Eq. 1 */
} hegrid_opts;

/* Non-finite sample values (NaN, +-Inf; flagged spectra are common in single-dish data).
 * PROPAGATE (default): IEEE arithmetic in Eq. 1 -- every cell within R of the sample gets
 *       NaN (or +-Inf) in that channel, as the fp64 definition does.
 * MASK: the value is missing: it is left out of both sums of its channel,
 *       V_c = sum_{n: v_cn finite} w v_cn / sum_{n: v_cn finite} w, NaN where no finite value
 *       remains; weight_map stays the channel-independent W = sum_n w (NEXT-4, SURVEY.md
 *       8(f)).  The cells affected by a masked value are recomputed after the launch. */
typedef enum hegrid_nonfinite {
    HEGRID_NONFINITE_PROPAGATE = 0,
    HEGRID_NONFINITE_MASK = 1
} hegrid_nonfinite;

/* Spatial index of a plan (the LUT of PAPER.md:177-192, sec. 3.1.1, Fig. 4/5).
 * BINS: map-aligned lon/lat bins, one per cell (rows of bins are contiguous sample ranges);
 *       feeds the tensor-core and SIMT engines; fields reaching within ~1 degree of a pole,
 *       spanning >= 180 degrees of longitude or with R > 1 degree are HEGRID_EUNSUPPORTED.
 * HEALPIX: the paper's own index: samples sorted by HEALPix ring-scheme pixel (Gorski et
 *       al. 2005); a cell gathers ring by ring over the pixel ranges that can
 *       reach it (Algorithm 1) with an fp64 distance test and fp64 sums.
 *       Any field, including polar caps and the whole sky; one gather kernel (the engine
 *       option is ignored).
 * AUTO: BINS where supported, else HEALPIX. */
typedef enum hegrid_index {
    HEGRID_INDEX_AUTO = 0,
    HEGRID_INDEX_BINS = 1,
    HEGRID_INDEX_HEALPIX = 2
} hegrid_index;

/* Value layouts accepted by hegrid_grid_device / hegrid_permute_device. */
typedef enum hegrid_layout {
    HEGRID_LAYOUT_USER_CN = 0,  /* [C][ld] fp32, sample s of channel c at c*ld + s, original
                                   sample order (the caller's natural layout) */
    HEGRID_LAYOUT_PLAN_NC = 1   /* [n_used][ld] fp32, channel c of plan position p at p*ld + c,
                                   plan (bin-sorted) order, channels contiguous: the hot
                                   loop's layout.  ld % 4 == 0 and 16-byte alignment required */
} hegrid_layout;

typedef struct hegrid_plan_s* hegrid_plan_t;

typedef struct hegrid_plan_stats {
    int64_t n_samples;          /* N given to the plan */
    int64_t n_used;             /* samples that can reach some cell (the rest are dropped) */
    int64_t n_bins;             /* bins of the spatial index (nrow * ncol) */
    int64_t n_candidate_pairs;  /* sum over cells of candidate-range lengths (superset) */
    int64_t n_pairs;            /* sum over cells of |{n : d <= R}| */
    int32_t nbr_min, nbr_max;   /* neighbours per cell */
    double nbr_mean;
    double t_plan_ms;           /* device time of plan construction */
    int32_t nrow, ncol;         /* bin grid (cells + margins) */
    int32_t mlat, mlon;         /* margins in bins */
    double sigma_deg, radius_deg;
    int64_t weight_image_bytes; /* device bytes of the precomputed weight image (0 = none) */
    int64_t tc_entries;         /* tensor-core engine schedule entries (0 = schedule not built
                                   yet: it is built by the first tensor-core launch) */
    int64_t tc_block_slots;     /* (entry, in-reach 4x4-cell block) pairs: each is one
                                   16-cell x 32-sample slot of the dense MMA product, so
                                   n_pairs / (512 tc_block_slots) is the useful MMA density */
    int32_t index;              /* hegrid_index the plan was built with (BINS or HEALPIX) */
    int32_t nside;              /* HEALPIX: HEALPix resolution parameter (0 for BINS) */
} hegrid_plan_stats;

/* ---- plan: spatial index (PAPER.md:177-192 steps 1,2,4; Algorithm 1 region lookup) ----
 * Sorts the samples into map-aligned bins (radix sort, stable: equal bins keep original
 * order), reorders coordinates, builds bin_start[] (the LUT).  lon_deg/lat_deg: host
 * [n] arrays.  n == 0 is legal (all-blank maps).  Errors: EINVAL, EDOMAIN, EUNSUPPORTED,
 * ENOMEM, ECUDA.  *out is set only on success. */
hegrid_status hegrid_plan_create(const double* lon_deg, const double* lat_deg, int64_t n,
                                 const hegrid_map* map, const hegrid_kernel* kernel,
                                 const hegrid_opts* opts, hegrid_plan_t* out);

/* Same, with device-resident coordinates (device pointers on opts->device); the work is
 * ordered on `stream` (cudaStream_t, NULL = legacy default) and the call returns after it
 * completes (validation result needed). */
hegrid_status hegrid_plan_create_device(const double* d_lon_deg, const double* d_lat_deg,
                                        int64_t n, const hegrid_map* map,
                                        const hegrid_kernel* kernel, const hegrid_opts* opts,
                                        void* stream, hegrid_plan_t* out);

/* Frees the plan and its device memory.  NULL is a no-op. */
void hegrid_plan_destroy(hegrid_plan_t plan);

/* Statistics; computes the pair counts on first call (one extra device pass). */
hegrid_status hegrid_plan_info(hegrid_plan_t plan, hegrid_plan_stats* out);

/* Per-sample weights (NEXT-4; reading R25): omega[n] >= 0 multiplies sample n's kernel
 * weight, w = omega_n w(d), so V = sum omega w v / sum omega w and W = sum omega w (e.g.
 * inverse noise variances of the spectra).  omega: host array of the
 * plan's n samples in original order, borrowed for the call; NULL restores omega = 1.  The
 * neighbour sets (hegrid_neighbours) stay geometric.  Drops the engine's per-plan tables
 * (they are rebuilt by the next grid call); the caller serialises it with the plan's other
 * calls.  Errors: EINVAL (n differs from the plan's), EDOMAIN (a weight non-finite or < 0),
 * ECUDA, ENOMEM. */
hegrid_status hegrid_plan_set_sample_weights(hegrid_plan_t plan, const float* omega, int64_t n);

/* Plan order: perm[p] = original index of the sample at plan position p, p < n_used
 * (host array of n_used entries; *n_used may be NULL). */
hegrid_status hegrid_plan_permutation(hegrid_plan_t plan, int64_t* perm, int64_t* n_used);

/* ---- grid: Eq. 1 for C channels, host buffers (end-to-end path) ----
 * data: host [C][N] fp32, original sample order (N = plan's n_samples).
 * out_map: host [C][ny][nx] fp32.  weight_map: host [ny][nx] fp32 (W), may be NULL.
 * Channel blocks are pipelined over opts->n_streams CUDA streams: H2D of block b,
 * device permute into plan order, accumulate + normalise, D2H, overlapping across
 * blocks.  Blocking: returns when out_map is complete.
 * C == 0 is a no-op (weight_map still written). */
hegrid_status hegrid_grid(hegrid_plan_t plan, const float* data, int64_t n_channels,
                          float* out_map, float* weight_map);

/* ---- grid on device buffers (the HBM-resident hot path) ----
 * d_data: device, layout per `layout` (hegrid_layout) with row stride ld (elements).
 * d_out: device [C][ny][nx] fp32; d_weight: device [ny][nx] or NULL.
 * Enqueued on `stream` (cudaStream_t); asynchronous.  USER_CN input is permuted through
 * a device scratch taken from the plan's stream-ordered pool on `stream` (extra HBM
 * traffic), so calls on different streams never share it.
 * Non-finite values (NaN, +-Inf; reading R15): the cells within R of such a sample get
 * the IEEE result of Eq. 1's sum (NaN, or +-Inf), exactly like the fp64 definition; all
 * other cells are unaffected.  |values| >= 2^128 (1 - 2^-12) count as +-Inf. */
hegrid_status hegrid_grid_device(hegrid_plan_t plan, const float* d_data, int64_t n_channels,
                                 int64_t ld, int32_t layout, float* d_out, float* d_weight,
                                 void* stream);

/* Device permute of user-order values into the plan layout (paper step 3):
 *   d_plan[p * ld_plan + c] = d_user[c * ld_user + perm[p]],  p < n_used, c < C.
 * ld_plan % 4 == 0.  Asynchronous on `stream`. */
hegrid_status hegrid_permute_device(hegrid_plan_t plan, const float* d_user, int64_t n_channels,
                                    int64_t ld_user, float* d_plan, int64_t ld_plan, void* stream);

/* Neighbour sets of cells [cell_begin, cell_end) (linear j*nx+i): Algorithm 1's gather set
 * {n : d(cell, s_n) <= R} (line "if d(target_cell[], raw_data[i]) <= R"),
 * enumerated on the device from the very pairs the plan's engine accumulates: for the
 * tensor-core engine (AUTO / TC) its per-tile chunk schedule and its weight expression
 * (a pair counts iff its weight is > 0), for the SIMT engine its per-cell candidate ranges
 * and predicate.  A pair the engine misses is missing here too, so comparing this set with
 * the fp64 definition checks the hot path's gather.  offsets: host
 * [cell_end-cell_begin+1]; sample_idx: host CSR of original sample indices, ascending
 * within each cell; NULL = counts only.  Blocking.  Errors: EINVAL (range), ECUDA, ENOMEM. */
hegrid_status hegrid_neighbours(hegrid_plan_t plan, int64_t cell_begin, int64_t cell_end,
                                int64_t* offsets, int64_t* sample_idx);

/* Stable LSD radix sort used by the plan, exposed for testing: perm = stable argsort of
 * host keys[n] (u32), computed on device `device`.  Blocking. */
hegrid_status hegrid_sort_u32(const uint32_t* keys, int64_t n, int32_t* perm, int32_t device);

/* HEALPix ring-scheme pixel index of n directions (the plan's HEALPIX key, computed on the
 * device with the same code): pix[k] = ang2pix_ring(nside, theta[k], phi[k]), theta the
 * colatitude in [0, pi] and phi the longitude in radians (any value; taken modulo 2 pi).
 * Host arrays of n elements, borrowed for the call.  nside a power of two in [1, 8192];
 * returns HEGRID_EINVAL otherwise, HEGRID_EDOMAIN for a non-finite or out-of-range theta.
 * Exposed so the index can be checked against an independent implementation. */
hegrid_status hegrid_healpix_ang2pix(int32_t nside, const double* theta, const double* phi,
                                     int64_t n, int64_t* pix, int32_t device);

/* Kernel-time profiling of the accumulate kernel: when enabled, hegrid_grid_device
 * brackets each accumulate launch with CUDA events on the caller's stream;
 * hegrid_profile_read synchronises, returns the summed milliseconds and launch count
 * since the last read, and resets them. */
hegrid_status hegrid_profile_enable(hegrid_plan_t plan, int32_t enable);
hegrid_status hegrid_profile_read(hegrid_plan_t plan, double* ms, int64_t* launches);

/* Pipeline trace of the last hegrid_grid call made while profiling was enabled
 * (hegrid_profile_enable): one row of 5 doubles per channel block,
 *   {slot (stream index), h2d_start, h2d_end, compute_end, d2h_end},
 * times in ms from the call's first event, from CUDA events recorded on each slot's stream
 * around the block's H2D copy, its device permute + accumulate (+ fix-up) and its D2H copy
 * (the paper's T2 / T3 / T4 stages, overlapped across streams as in
 * :279-294).  buf: host [cap_rows][5] or NULL (count only); *n_rows = rows available. */
hegrid_status hegrid_pipeline_trace(hegrid_plan_t plan, double* buf, int64_t cap_rows,
                                    int64_t* n_rows);

/* Number of kernels this library has launched in this process (all plans). */
int64_t hegrid_launch_count(void);

/* Static string for a status code. */
const char* hegrid_status_string(hegrid_status s);

/* HEGRID_ABI_VERSION of the loaded library. */
int32_t hegrid_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HEGRID_H */
