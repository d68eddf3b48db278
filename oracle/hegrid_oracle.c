/*
 * hegrid_oracle.c -- fp64 brute-force CPU oracle for HEGrid's gridding (Eq. 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2207_04584_b200/) never links, imports or calls it, and it shares no code,
 * header, constant or helper with the CUDA path.
 *
 * What it computes (Sec. 2.2, Eq. 1):
 *     V[g_ij] = (1 / W_ij) * sum_n V[s_n] * w(a_ij, d_ij; a_n, d_n),   W_ij = sum_n w(...)
 * with the readings listed in DESIGN.md "Readings of the paper":
 *   - w is a Gaussian of the great-circle distance d (R1):
 *         w = exp(-d^2 / (2 sigma^2)) for d <= R, else 0,
 *     sigma = FWHM / (2 sqrt(2 ln 2)) (R2), R = support * sigma (R3, default 3).
 *   - the support test is inclusive, d <= R, as in Algorithm 1 line
 *     "if d(target_cell[], raw_data[i]) <= R" (R4).
 *   - d is the haversine great-circle distance in fp64 (R5):
 *         h = sin^2(dlat/2) + cos(lat_c) cos(lat_n) sin^2(dlon/2),  d = 2 asin(min(1, sqrt h)),
 *     dlon wrapped to (-180, 180] degrees (R9).
 *   - cell (i, j) centre, 0-based i (lon, fastest) and j (lat) (R6):
 *         lon = crval_lon + (i + 1 - crpix_x) * cdelt_lon,
 *         lat = crval_lat + (j + 1 - crpix_y) * cdelt_lat.
 *   - W = 0 gives V = NaN (R8); the weight map keeps W.
 *   - sums run over samples in ascending original index, in fp64 (R12).
 *
 * Structure follows the plain definition: for every requested cell, test every
 * sample (no index, no pruning, no blocking), collect the neighbour list in
 * ascending sample order, then for every requested channel sum w * v over that
 * list.  OpenMP only splits the outer loop over cells; each cell is computed by
 * one thread in a fixed order, so results do not depend on the thread count.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Map header: the oracle's own copy (it includes no product header). */
typedef struct {
    int32_t nx, ny;
    double crval_lon, crval_lat;
    double crpix_x, crpix_y;
    double cdelt_lon, cdelt_lat;
    int32_t projection;     /* 0 linear lon/lat (R6), 1 TAN, 2 SIN (reading R26) */
    int32_t reserved;
} ora_map;

static const double ORA_PI = 3.14159265358979323846;

static double deg2rad(double x) { return x * (ORA_PI / 180.0); }

/* sigma from the kernel FWHM: FWHM = 2 sqrt(2 ln 2) sigma (reading R2). */
double ora_sigma_deg(double fwhm_deg) { return fwhm_deg / (2.0 * sqrt(2.0 * log(2.0))); }

/* Wrap a longitude difference (degrees) into (-180, 180] (reading R9). */
double ora_wrap180(double x) {
    double y = fmod(x, 360.0);          /* (-360, 360) */
    if (y > 180.0) y -= 360.0;
    if (y <= -180.0) y += 360.0;
    return y;
}

/* Cell centre of 0-based cell (i, j).  Linear lon/lat grid (reading R6), or a zenithal
 * projection (reading R26) written as in the FITS WCS definition (Calabretta & Greisen
 * 2002, A&A 395, 1077): intermediate world coordinates x, y (deg); native longitude
 * phi = arg(-y, x) (their eq. 14); native latitude theta = atan(180/pi / R) for TAN (eq. 54)
 * or acos(pi/180 R) for SIN (eq. 59, R = sqrt(x^2 + y^2)); native -> celestial with the
 * native pole at (crval_lon, crval_lat) and LONPOLE phi_p = 180 deg (eq. 2). */
void ora_cell_centre(const ora_map* m, int64_t i, int64_t j, double* lon, double* lat) {
    double x = ((double)i + 1.0 - m->crpix_x) * m->cdelt_lon;
    double y = ((double)j + 1.0 - m->crpix_y) * m->cdelt_lat;
    if (m->projection == 0) {
        *lon = m->crval_lon + x;
        *lat = m->crval_lat + y;
        return;
    }
    double r = sqrt(x * x + y * y);
    double phi = (r == 0.0) ? 0.0 : atan2(x, -y);
    double theta;
    if (m->projection == 1) {
        theta = atan2(180.0 / ORA_PI, r);
    } else {
        double a = r * ORA_PI / 180.0;
        theta = a <= 1.0 ? acos(a) : NAN;
    }
    double ap = deg2rad(m->crval_lon), dp = deg2rad(m->crval_lat), php = ORA_PI;
    double sd = sin(theta) * sin(dp) + cos(theta) * cos(dp) * cos(phi - php);
    if (sd > 1.0) sd = 1.0;
    if (sd < -1.0) sd = -1.0;
    double a = ap + atan2(-cos(theta) * sin(phi - php),
                          sin(theta) * cos(dp) - cos(theta) * sin(dp) * cos(phi - php));
    *lat = asin(sd) * 180.0 / ORA_PI;
    *lon = a * 180.0 / ORA_PI;
}

/* Great-circle distance in radians, haversine form (reading R5). */
double ora_distance_rad(double lon1, double lat1, double lon2, double lat2) {
    double dlon = deg2rad(ora_wrap180(lon2 - lon1));
    double dlat = deg2rad(lat2 - lat1);
    double s1 = sin(0.5 * dlat);
    double s2 = sin(0.5 * dlon);
    double h = s1 * s1 + cos(deg2rad(lat1)) * cos(deg2rad(lat2)) * (s2 * s2);
    double r = sqrt(h);
    if (r > 1.0) r = 1.0;
    return 2.0 * asin(r);
}

double ora_distance_deg(double lon1, double lat1, double lon2, double lat2) {
    return ora_distance_rad(lon1, lat1, lon2, lat2) * (180.0 / ORA_PI);
}

/* Gaussian kernel of Eq. 1 with inclusive support test (readings R1, R3, R4).
 * d, sigma, R in radians.  Returns 0 outside the support. */
double ora_weight(double d, double sigma, double R) {
    if (!(d <= R)) return 0.0;
    return exp(-(d * d) / (2.0 * sigma * sigma));
}

/* Tophat kernel (KernelSpec kind "tophat": 1 for d <= R, else 0). */
double ora_weight_tophat(double d, double R) {
    return (d <= R) ? 1.0 : 0.0;
}

/* Neighbour list of one cell: every sample n (ascending) with d <= R.
 * Returns the count; writes idx/w if non-NULL. */
static int64_t cell_neighbours(const double* lon, const double* lat, int64_t n,
                               double lon_c, double lat_c, double sigma, double R, int kind,
                               int64_t* idx, double* w) {
    int64_t k = 0;
    for (int64_t s = 0; s < n; ++s) {
        double d = ora_distance_rad(lon_c, lat_c, lon[s], lat[s]);
        if (d <= R) {
            if (idx) idx[k] = s;
            if (w) w[k] = kind == 1 ? ora_weight_tophat(d, R) : ora_weight(d, sigma, R);
            ++k;
        }
    }
    return k;
}

static int valid_inputs(const ora_map* m, double fwhm, double support, int64_t n) {
    if (!m || m->nx < 1 || m->ny < 1 || n < 0) return 0;
    if (!(fwhm > 0.0) || !(support > 0.0)) return 0;
    return 1;
}

/*
 * Eq. 1 on a set of cells and a set of channels.
 *   lon, lat   [n] degrees
 *   vals       channel c's value of sample s is vals[c * ld + s] (float32, widened to fp64)
 *   ch_idx     [n_ch] channels to grid (NULL = 0..n_ch-1)
 *   cell_idx   [n_cells] linear cell indices j*nx + i (NULL = all cells, n_cells = nx*ny)
 *   out        [n_ch][n_cells] normalised values (NaN where W = 0); may be NULL
 *   wsum       [n_cells] W; may be NULL
 *   nbr_count  [n_cells] number of samples with d <= R; may be NULL
 *   nthreads   OpenMP threads (<= 0: runtime default)
 *   kind       0 = Gaussian (Eq. 1's kernel, readings R1-R3), 1 = tophat
 *   sample_w   [n] per-sample weights omega_s >= 0 multiplying the kernel weight (NEXT-4,
 *              DESIGN.md reading R25: w = omega_s w(d), W = sum_s omega_s w(d)); NULL = 1
 *   mask       0: non-finite values enter the sums with IEEE semantics (reading R15);
 *              1: a non-finite value is missing: it leaves both sums of its channel,
 *              V_c = sum_{finite} w v / sum_{finite} w (reading R24); W stays sum_s w
 * Returns 0 on success, 1 on invalid arguments, 3 on allocation failure.
 */
int ora_grid_cells_ex(const double* lon, const double* lat, int64_t n,
                      const float* vals, int64_t ld, const int64_t* ch_idx, int64_t n_ch,
                      const ora_map* m, double fwhm_deg, double support,
                      const int64_t* cell_idx, int64_t n_cells,
                      double* out, double* wsum, int64_t* nbr_count, int nthreads, int kind,
                      const double* sample_w, int mask) {
    if (!valid_inputs(m, fwhm_deg, support, n)) return 1;
    if (kind != 0 && kind != 1) return 1;
    if (mask != 0 && mask != 1) return 1;
    if (n_ch < 0 || (n_ch > 0 && !vals) || (n > 0 && (!lon || !lat))) return 1;
    int64_t ncell_all = (int64_t)m->nx * (int64_t)m->ny;
    if (!cell_idx) n_cells = ncell_all;
    double sigma = deg2rad(ora_sigma_deg(fwhm_deg));
    double R = support * sigma;
    int failed = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
        double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        if (!idx || !w) {
#pragma omp atomic write
            failed = 1;
        }
#pragma omp for schedule(dynamic, 4)
        for (int64_t q = 0; q < n_cells; ++q) {
            if (!idx || !w) continue;
            int64_t cell = cell_idx ? cell_idx[q] : q;
            int64_t i = cell % m->nx, j = cell / m->nx;
            double lon_c, lat_c;
            ora_cell_centre(m, i, j, &lon_c, &lat_c);
            int64_t k = cell_neighbours(lon, lat, n, lon_c, lat_c, sigma, R, kind, idx, w);
            if (sample_w)
                for (int64_t t = 0; t < k; ++t) w[t] *= sample_w[idx[t]];
            double W = 0.0;
            for (int64_t t = 0; t < k; ++t) W += w[t];
            if (wsum) wsum[q] = W;
            if (nbr_count) nbr_count[q] = k;
            if (out) {
                for (int64_t c = 0; c < n_ch; ++c) {
                    int64_t ch = ch_idx ? ch_idx[c] : c;
                    const float* row = vals + ch * ld;
                    double S = 0.0, Wc = 0.0;
                    for (int64_t t = 0; t < k; ++t) {
                        double v = (double)row[idx[t]];
                        if (mask && !isfinite(v)) continue;
                        S += w[t] * v;
                        Wc += w[t];
                    }
                    double Wv = mask ? Wc : W;
                    out[c * n_cells + q] = (Wv > 0.0) ? S / Wv : NAN;
                }
            }
        }
        free(idx);
        free(w);
    }
    return failed ? 3 : 0;
}

int ora_grid_cells(const double* lon, const double* lat, int64_t n,
                   const float* vals, int64_t ld, const int64_t* ch_idx, int64_t n_ch,
                   const ora_map* m, double fwhm_deg, double support,
                   const int64_t* cell_idx, int64_t n_cells,
                   double* out, double* wsum, int64_t* nbr_count, int nthreads, int kind) {
    return ora_grid_cells_ex(lon, lat, n, vals, ld, ch_idx, n_ch, m, fwhm_deg, support, cell_idx,
                             n_cells, out, wsum, nbr_count, nthreads, kind, NULL, 0);
}

/*
 * Neighbour sets (Algorithm 1's "d(target_cell, raw_data[i]) <= R" set) as CSR.
 *   offsets [n_cells + 1]; idx [offsets[n_cells]] ascending original sample index,
 *   idx may be NULL to count only.  cell_idx NULL = all cells.
 */
int ora_neighbours(const double* lon, const double* lat, int64_t n, const ora_map* m,
                   double fwhm_deg, double support, const int64_t* cell_idx, int64_t n_cells,
                   int64_t* offsets, int64_t* idx, int nthreads) {
    if (!valid_inputs(m, fwhm_deg, support, n) || !offsets) return 1;
    if (!cell_idx) n_cells = (int64_t)m->nx * (int64_t)m->ny;
    double sigma = deg2rad(ora_sigma_deg(fwhm_deg));
    double R = support * sigma;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    /* pass 1: counts */
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < n_cells; ++q) {
        int64_t cell = cell_idx ? cell_idx[q] : q;
        double lon_c, lat_c;
        ora_cell_centre(m, cell % m->nx, cell / m->nx, &lon_c, &lat_c);
        offsets[q + 1] = cell_neighbours(lon, lat, n, lon_c, lat_c, sigma, R, 0, NULL, NULL);
    }
    offsets[0] = 0;
    for (int64_t q = 0; q < n_cells; ++q) offsets[q + 1] += offsets[q];
    if (!idx) return 0;
    /* pass 2: fill */
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t q = 0; q < n_cells; ++q) {
        int64_t cell = cell_idx ? cell_idx[q] : q;
        double lon_c, lat_c;
        ora_cell_centre(m, cell % m->nx, cell / m->nx, &lon_c, &lat_c);
        cell_neighbours(lon, lat, n, lon_c, lat_c, sigma, R, 0, idx + offsets[q], NULL);
    }
    return 0;
}

int ora_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
