// healpix.cuh -- HEALPix ring-scheme pixelisation (Gorski et al. 2005, ApJ 622, 759), the
// pixelisation of the paper's LUT (sec. 3.1.1 and its footnote; Fig. 4:
// "Each pixel has its index information, including pixel_idx, ring_idx, ring length").
// Written from the published ring-scheme layout (SPEC.md:17-110 restates it):
//   npix = 12 nside^2, rings i = 1 .. 4 nside - 1;
//   north cap  i <  nside : 4 i pixels from 2 i (i - 1),      z = 1 - i^2 / (3 nside^2),
//                           pixel centres phi_j = (j + 1/2) 2 pi / (4 i);
//   equatorial nside <= i <= 3 nside : 4 nside pixels from 2 nside (nside - 1) +
//                           (i - nside) 4 nside, z = 4/3 - 2 i / (3 nside), pixel centres
//                           phi_j = (j + f) 2 pi / (4 nside), f = 0 if i + nside is odd,
//                           f = 1/2 if it is even (every other ring is shifted);
//   south cap mirrors the north cap.
// All functions are fp64 and usable on host and device.
#pragma once

#include <math.h>
#include <stdint.h>

namespace hg {
namespace hpx {

struct Ring {
    int64_t start;   // first pixel
    int64_t len;     // pixels on the ring
    double z;        // cos(colatitude) of the ring centre
    double f;        // pixel j's centre is at phi = (j + f) 2 pi / len
};

__host__ __device__ inline int64_t npix(int64_t nside) { return 12 * nside * nside; }
__host__ __device__ inline int nrings(int64_t nside) { return (int)(4 * nside - 1); }

__host__ __device__ inline Ring ring_info(int64_t nside, int i) {
    Ring r;
    const int64_t ncap = 2 * nside * (nside - 1);
    if (i < nside) {                          // north polar cap
        r.len = 4 * (int64_t)i;
        r.start = 2 * (int64_t)i * (i - 1);
        r.z = 1.0 - (double)i * i / (3.0 * nside * nside);
        r.f = 0.5;
    } else if (i <= 3 * nside) {              // equatorial belt
        r.len = 4 * nside;
        r.start = ncap + (int64_t)(i - nside) * 4 * nside;
        r.z = (4.0 / 3.0) - 2.0 * i / (3.0 * nside);
        r.f = ((i + nside) & 1) ? 0.0 : 0.5;
    } else {                                  // south polar cap
        const int ii = (int)(4 * nside - i);
        r.len = 4 * (int64_t)ii;
        r.start = npix(nside) - 2 * (int64_t)ii * (ii + 1);
        r.z = -1.0 + (double)ii * ii / (3.0 * nside * nside);
        r.f = 0.5;
    }
    return r;
}

// colatitude of ring i's centre, with ring 0 = the north pole and ring 4 nside = the south pole
__host__ __device__ inline double ring_theta(int64_t nside, int i) {
    if (i <= 0) return 0.0;
    if (i >= 4 * nside) return M_PI;
    const double z = ring_info(nside, i).z;
    if (fabs(z) < 0.99) return acos(z);
    // near the poles: theta = 2 asin(sqrt((1 - |z|) / 2)), 1 - |z| = i'^2 / (3 nside^2) exactly
    const int ii = i < nside ? i : (int)(4 * nside - i);
    const double t = 2.0 * asin(sqrt((double)ii * ii / (6.0 * nside * nside)));
    return z > 0 ? t : M_PI - t;
}

// ang2pix_ring: the pixel containing the direction (colatitude theta in [0, pi], longitude
// phi in radians, any value).  The equatorial branch locates the pixel between the two
// families of edge lines phi / (pi/2) +- 3 z / 4 = const; the caps use the radial coordinate
// nside sqrt(3 (1 - |z|)) = nside sqrt(6) sin(theta'/2), theta' the distance to the nearest
// pole (the form that stays accurate at the pole).
__host__ __device__ inline int64_t ang2pix_ring(int64_t nside, double theta, double phi) {
    const double z = cos(theta), za = fabs(z);
    double tt = fmod(phi * (2.0 / M_PI), 4.0);          // phi in units of pi/2, in [0, 4)
    if (tt < 0) tt += 4.0;
    if (tt >= 4.0) tt = 0.0;
    const int64_t nl4 = 4 * nside;
    if (za <= 2.0 / 3.0) {
        const double t1 = nside * (0.5 + tt), t2 = nside * z * 0.75;
        const int64_t jp = (int64_t)floor(t1 - t2);      // ascending edge line index
        const int64_t jm = (int64_t)floor(t1 + t2);      // descending edge line index
        const int64_t ir = nside + 1 + jp - jm;          // ring from z = 2/3, in [1, 2 nside + 1]
        const int64_t kshift = 1 - (ir & 1);
        const int64_t t = jp + jm - nside + kshift + 1 + 2 * nl4;   // kept positive before the halving
        const int64_t ip = (t >> 1) % nl4;
        return 2 * nside * (nside - 1) + (ir - 1) * nl4 + ip;
    }
    const double tp = tt - floor(tt);
    const double th = z > 0 ? theta : M_PI - theta;     // distance to the nearest pole
    const double tmp = nside * sqrt(6.0) * sin(0.5 * th);
    int64_t jp = (int64_t)floor(tp * tmp), jm = (int64_t)floor((1.0 - tp) * tmp);
    int64_t ir = jp + jm + 1;                            // ring from the nearest pole
    if (ir > nside) ir = nside;                          // |z| = 2/3 edge case
    if (ir < 1) ir = 1;
    int64_t ip = (int64_t)floor(tt * ir);
    ip = ((ip % (4 * ir)) + 4 * ir) % (4 * ir);
    return z > 0 ? 2 * ir * (ir - 1) + ip : npix(nside) - 2 * ir * (ir + 1) + ip;
}

// pix2ang_ring: centre of pixel p (colatitude, longitude in [0, 2 pi))
__host__ __device__ inline void pix2ang_ring(int64_t nside, int64_t p, double* theta, double* phi) {
    // ring of p by bisection over ring starts (rings are few; keeps one definition of the layout)
    int lo = 1, hi = nrings(nside);
    while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (ring_info(nside, mid).start <= p) lo = mid; else hi = mid - 1;
    }
    const Ring r = ring_info(nside, lo);
    *theta = ring_theta(nside, lo);
    *phi = ((double)(p - r.start) + r.f) * (2.0 * M_PI / (double)r.len);
}

// ring_above(z): the ring directly north of z (0 if z is north of ring 1)
__host__ __device__ inline int ring_above(int64_t nside, double theta) {
    const double z = cos(theta), az = fabs(z);
    if (az <= 2.0 / 3.0) return (int)floor(nside * (2.0 - 1.5 * z));
    const double th = z > 0 ? theta : M_PI - theta;
    const int ir = (int)floor(nside * sqrt(6.0) * sin(0.5 * th));
    return z > 0 ? ir : (int)(4 * nside - ir - 1);
}

// The pixel intervals of ring i that can hold a sample within radius R of the direction
// (theta_c, phi_c) (Algorithm 1's "min / max contribution pixel"),
// conservatively: a sample in ring i's pixels lies between the centres of rings i - 1 and
// i + 1; within R of the centre its longitude offset obeys sin|dphi| <= sin R / sin(theta)
// (spherical sine law; |dphi| <= pi/2 when the cap holds no pole); pixels are taken with
// their centres within that offset plus two pixel widths (a pixel's longitude extent around
// its centre is below one width).  Returns the number of intervals (0, 1 or 2) in
// [p0[k], p1[k]] (inclusive pixel indices).
__host__ __device__ inline int ring_query(int64_t nside, int i, double theta_c, double phi_c,
                                          double R, bool pole_cap, int64_t p0[2], int64_t p1[2]) {
    const Ring r = ring_info(nside, i);
    const double tlo = fmax(theta_c - R, 0.0), thi = fmin(theta_c + R, M_PI);
    const double ta = fmax(ring_theta(nside, i - 1), tlo), tb = fmin(ring_theta(nside, i + 1), thi);
    if (ta > tb) return 0;
    bool full = pole_cap;
    double dphi = M_PI;
    if (!full) {
        const double smin = fmin(sin(ta), sin(tb));
        const double q = smin > 1e-12 ? sin(R) / smin : 2.0;
        if (q >= 1.0) full = true; else dphi = asin(q);
    }
    if (!full) {
        const double w = 2.0 * M_PI / (double)r.len;
        const double a = (phi_c - dphi) / w - r.f - 2.0, b = (phi_c + dphi) / w - r.f + 2.0;
        const int64_t jlo = (int64_t)ceil(a), jhi = (int64_t)floor(b);
        if (jhi - jlo + 1 >= r.len) {
            full = true;
        } else {
            const int64_t l0 = ((jlo % r.len) + r.len) % r.len;
            const int64_t n = jhi - jlo + 1;
            if (l0 + n <= r.len) {
                p0[0] = r.start + l0;
                p1[0] = r.start + l0 + n - 1;
                return 1;
            }
            p0[0] = r.start + l0;
            p1[0] = r.start + r.len - 1;
            p0[1] = r.start;
            p1[1] = r.start + (l0 + n - r.len) - 1;
            return 2;
        }
    }
    p0[0] = r.start;
    p1[0] = r.start + r.len - 1;
    return 1;
}

// smallest power-of-two nside with mean pixel spacing sqrt(4 pi / npix) <= spacing (rad),
// in [1, 8192] (spacing = min(cell size, R) / 2)
inline int choose_nside(double spacing) {
    int ns = 1;
    while (ns < 8192 && sqrt(4.0 * M_PI / (12.0 * ns * (double)ns)) > spacing) ns *= 2;
    return ns;
}

}  // namespace hpx
}  // namespace hg
