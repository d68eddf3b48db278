"""Pins for the fp64 oracle against things other than itself (closed forms, invariants,
an independent library).  Each pin is chosen so that a plausible slip in the oracle --
a dropped cos(lat) factor, a wrong sign or index, a transposed operand, a wrong
sigma, an exclusive instead of inclusive support test, a missing normalisation --
fails at least one test.  Citations: PAPER.md:135-148 (Eq. 1)
(Algorithm 1 support test), SPEC.md lines as quoted, readings R1-R18.
"""
import math
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
FWHM2SIG = 2.0 * math.sqrt(2.0 * math.log(2.0))


def unit(lon, lat):
    lo, la = np.radians(lon), np.radians(lat)
    return np.stack([np.cos(la) * np.cos(lo), np.cos(la) * np.sin(lo), np.sin(la)], -1)


def dist_atan2(lon1, lat1, lon2, lat2):
    """Great-circle distance (rad) via atan2(|u x v|, u.v): a formula independent of
    the oracle's haversine, accurate at all separations."""
    u, v = unit(lon1, lat1), unit(lon2, lat2)
    return np.arctan2(np.linalg.norm(np.cross(u, v), axis=-1), np.sum(u * v, -1))


def mk_map(nx, ny, lon0, lat0, d_lon, d_lat=None):
    return dict(nx=nx, ny=ny, crval_lon=lon0, crval_lat=lat0, crpix_x=(nx + 1) / 2,
                crpix_y=(ny + 1) / 2, cdelt_lon=d_lon, cdelt_lat=d_lon if d_lat is None else d_lat)


def load_golden(name):
    rows = {}
    with open(os.path.join(HERE, "golden", name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                k, v = line.split("=", 1)
                rows[k.strip()] = [float(x) for x in v.split(",")]
    return rows


# ---------------------------------------------------------------- distance and kernel
def test_kernel_values_golden():
    """gaussian(sigma=1, R=3): d=0 -> 1, d=sigma -> exp(-0.5), d=3.1 -> 0."""
    g = load_golden("kernel_values.txt")
    s, R = math.radians(1.0), math.radians(3.0)
    assert oracle.weight(0.0, s, R) == 1.0
    assert oracle.weight(math.radians(1.0), s, R) == pytest.approx(g["w_at_sigma"][0], rel=1e-10)
    assert oracle.weight(math.radians(3.1), s, R) == 0.0
    # inclusive support ("<= R")
    assert oracle.weight(R, s, R) == pytest.approx(math.exp(-4.5), rel=1e-15)
    # sigma from FWHM (reading R2): FWHM = 2 sqrt(2 ln 2) sigma
    assert oracle.sigma_deg(g["fwhm_deg"][0]) == pytest.approx(g["sigma_deg"][0], rel=1e-12)


def test_distance_golden_examples():
    """identity, 90 deg quarter circle, (10,40)-(11,40) ~ 0.766 deg."""
    g = load_golden("kernel_values.txt")
    assert oracle.distance_deg(12.0, 34.0, 12.0, 34.0) == 0.0
    assert oracle.distance_deg(0.0, 0.0, 90.0, 0.0) == pytest.approx(90.0, rel=1e-14)
    assert oracle.distance_deg(10, 40, 11, 40) == pytest.approx(g["d_10_40_11_40"][0], abs=1e-5)
    assert oracle.distance_deg(10, 40, 11, 40) == pytest.approx(
        math.degrees(dist_atan2(10, 40, 11, 40)), rel=1e-12)


def test_distance_matches_independent_formula_random_pairs():
    rng = np.random.default_rng(1)
    lon1 = rng.uniform(0, 360, 2000)
    lat1 = rng.uniform(-80, 80, 2000)
    # separations from 1e-6 deg to 60 deg, and across the lon wrap
    sep = 10 ** rng.uniform(-6, 1.8, 2000)
    ang = rng.uniform(0, 2 * np.pi, 2000)
    lat2 = np.clip(lat1 + sep * np.sin(ang), -89, 89)
    lon2 = (lon1 + sep * np.cos(ang) / np.cos(np.radians(lat1)) + 360) % 360
    got = np.array([oracle.distance_deg(a, b, c, d) for a, b, c, d in zip(lon1, lat1, lon2, lat2)])
    ref = np.degrees(dist_atan2(lon1, lat1, lon2, lat2))
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-13)


def test_lon_wrap():
    """Reading R9: longitude differences wrap; 359.9 and 0.1 are 0.2 deg apart on the equator."""
    assert oracle.wrap180(359.9 - 0.1) == pytest.approx(-0.2, abs=1e-12)
    assert oracle.wrap180(-180.0) == 180.0
    assert oracle.wrap180(180.0) == 180.0
    assert oracle.distance_deg(359.9, 0.0, 0.1, 0.0) == pytest.approx(0.2, rel=1e-10)


def test_cell_centres_follow_map_header():
    """Reading R6: lon = crval + (i+1-crpix)*cdelt, same for lat; crpix=(n+1)/2 centres the map."""
    m = mk_map(4, 3, 30.0, 41.0, -0.5, 0.25)
    assert oracle.cell_centre(m, 0, 0) == pytest.approx((30.0 + 1.5 * 0.5, 41.0 - 0.25))
    assert oracle.cell_centre(m, 3, 2) == pytest.approx((30.0 - 1.5 * 0.5, 41.0 + 0.25))


# ---------------------------------------------------------------- Eq. 1 closed forms
def test_centre_weight_is_one():
    """A sample bit-identical to a cell centre has d = 0 and w = exp(0) = 1 (north_star pin)."""
    m = mk_map(5, 5, 30.0, 41.0, 1.0 / 60)
    lon_c, lat_c = oracle.cell_centre(m, 2, 3)
    out, W, cnt = oracle.grid(np.array([lon_c]), np.array([lat_c]), np.array([[5.0]], np.float32),
                              m, 3.0 / 60)
    cell = 3 * 5 + 2
    assert W[cell] == 1.0
    assert out[0, cell] == 5.0
    assert cnt[cell] == 1


def test_single_sample_reproduces_kernel_profile_off_equator():
    """One sample: W(cell) = exp(-d^2/2 sigma^2) [d <= R] with d from the independent
    atan2 formula, and V = v on every covered cell.  At lat 41 deg this pins the
    cos(lat) factor of the distance."""
    m = mk_map(21, 21, 30.0, 41.0, 0.5 / 60)
    fwhm = 3.0 / 60
    sig = math.radians(fwhm / FWHM2SIG)
    R = 3.0 * sig
    lon_s, lat_s = 30.0013, 41.0021
    out, W, cnt = oracle.grid(np.array([lon_s]), np.array([lat_s]), np.array([[2.5]], np.float32),
                              m, fwhm)
    jj, ii = np.divmod(np.arange(21 * 21), 21)
    lon_c = 30.0 + (ii + 1 - 11) * (0.5 / 60)
    lat_c = 41.0 + (jj + 1 - 11) * (0.5 / 60)
    d = dist_atan2(lon_c, lat_c, lon_s, lat_s)
    ref = np.where(d <= R, np.exp(-d * d / (2 * sig * sig)), 0.0)
    np.testing.assert_allclose(W, ref, rtol=1e-10, atol=0)
    covered = ref > 0
    assert covered.sum() > 20 and (~covered).sum() > 20
    np.testing.assert_allclose(out[0, covered], 2.5, rtol=2e-16)
    assert np.all(np.isnan(out[0, ~covered]))
    # an exact lon-only offset at 41 deg: d is NOT the coordinate offset (cos factor)
    d_lon_only = dist_atan2(30.0, 41.0, 30.0 + 0.05, 41.0)
    assert abs(d_lon_only - math.radians(0.05)) > 0.2 * math.radians(0.05)


def test_support_edge_inclusive_and_nothing_beyond():
    """Equator: d = |dlon| exactly.  d = R(1 - 1e-9) contributes, d = R(1 + 1e-9) does not."""
    fwhm = 3.0 / 60
    R_deg = 3.0 * fwhm / FWHM2SIG
    m = mk_map(1, 1, 10.0, 0.0, 1.0 / 60)
    for f, inside in ((1 - 1e-9, True), (1 + 1e-9, False)):
        out, W, cnt = oracle.grid(np.array([10.0 + f * R_deg]), np.array([0.0]),
                                  np.array([[1.0]], np.float32), m, fwhm)
        assert (cnt[0] == 1) == inside
        if inside:
            assert W[0] == pytest.approx(math.exp(-4.5), rel=1e-6)
        else:
            assert W[0] == 0.0 and np.isnan(out[0, 0])
    # on a meridian d = |dlat|
    m2 = mk_map(1, 1, 10.0, 41.0, 1.0 / 60)
    for f, inside in ((1 - 1e-9, True), (1 + 1e-9, False)):
        _, _, cnt = oracle.grid(np.array([10.0]), np.array([41.0 - f * R_deg]),
                                np.array([[1.0]], np.float32), m2, fwhm)
        assert (cnt[0] == 1) == inside


def test_weight_sums_closed_form_equatorial_strip():
    """1-D Nadaraya-Watson on the equator: cells at i*D, samples at k*s,
    W_i = sum_k exp(-(iD - ks)^2 / 2 sigma^2) [|iD - ks| <= R] (north_star pin)."""
    nx = 9
    D = 1.0 / 60
    s_step = 0.37 / 60
    fwhm = 3.0 / 60
    sig_deg = fwhm / FWHM2SIG
    R_deg = 3.0 * sig_deg
    m = dict(nx=nx, ny=1, crval_lon=0.0, crval_lat=0.0, crpix_x=1.0, crpix_y=1.0,
             cdelt_lon=D, cdelt_lat=D)
    ks = np.arange(-20, 45)
    lon = ks * s_step
    lat = np.zeros_like(lon)
    vals = (1.0 + 0.25 * ks).astype(np.float32)[None, :]
    out, W, cnt = oracle.grid(lon, lat, vals, m, fwhm)
    for i in range(nx):
        dd = np.abs(i * D - ks * s_step)
        w = np.where(dd <= R_deg, np.exp(-dd ** 2 / (2 * sig_deg ** 2)), 0.0)
        assert W[i] == pytest.approx(w.sum(), rel=1e-10)
        assert cnt[i] == int((dd <= R_deg).sum())
        assert out[0, i] == pytest.approx((w * vals[0].astype(np.float64)).sum() / w.sum(), rel=1e-10)


def test_constant_input_gives_constant_map():
    """constant sky -> constant map on covered cells, blank elsewhere."""
    rng = np.random.default_rng(3)
    lon = 30 + rng.uniform(-0.1, 0.1, 3000)
    lat = 41 + rng.uniform(-0.1, 0.1, 3000)
    m = mk_map(24, 24, 30.0, 41.0, 0.5 / 60)
    c = np.float32(7.318)
    out, W, _ = oracle.grid(lon, lat, np.full((1, 3000), c, np.float32), m, 3.0 / 60)
    cov = W > 0
    assert cov.all()
    # SPEC.md:444 "within 1e-12": fp64 rounding of ~10^2-term sums only
    assert np.max(np.abs(out[0] - float(c))) <= 1e-12 * float(c)


def test_symmetric_samples_average():
    """samples 3 and 5 equidistant from a cell -> 4; four samples at
    +-delta in lon and lat on the equator (equal distances there) -> their mean."""
    m = mk_map(1, 1, 20.0, 0.0, 1.0 / 60)
    dl = 0.8 / 60
    out, _, _ = oracle.grid(np.array([20 - dl, 20 + dl]), np.array([0.0, 0.0]),
                            np.array([[3.0, 5.0]], np.float32), m, 3.0 / 60)
    assert out[0, 0] == pytest.approx(4.0, rel=1e-14)
    out, _, _ = oracle.grid(np.array([20 - dl, 20 + dl, 20, 20]), np.array([0, 0, -dl, dl]),
                            np.array([[1.0, 2.0, 3.0, 6.0]], np.float32), m, 3.0 / 60)
    assert out[0, 0] == pytest.approx(3.0, rel=1e-12)


def test_zero_samples_all_blank():
    """zero samples -> all NaN values, zero weights."""
    m = mk_map(4, 4, 0.0, 0.0, 0.1)
    out, W, cnt = oracle.grid(np.zeros(0), np.zeros(0), np.zeros((2, 0), np.float32), m, 0.3)
    assert np.all(np.isnan(out)) and np.all(W == 0) and np.all(cnt == 0)


def test_brute_force_tiny_instance_independent_distance():
    """Brute force on a tiny random instance with the independent atan2 distance:
    out = sum(w v)/sum(w) per cell and per channel (pins channel/sample indexing)."""
    rng = np.random.default_rng(11)
    N, C = 60, 3
    lon = 30 + rng.uniform(-0.06, 0.06, N)
    lat = 41 + rng.uniform(-0.06, 0.06, N)
    v = rng.normal(10, 2, (C, N)).astype(np.float32)
    m = mk_map(6, 5, 30.0, 41.0, 1.0 / 60, 1.2 / 60)
    fwhm = 3.0 / 60
    out, W, cnt = oracle.grid(lon, lat, v, m, fwhm)
    sig = math.radians(fwhm / FWHM2SIG)
    for j in range(5):
        for i in range(6):
            lc = 30 + (i + 1 - 3.5) / 60
            bc = 41 + (j + 1 - 3.0) * 1.2 / 60
            d = dist_atan2(lc, bc, lon, lat)
            w = np.where(d <= 3 * sig, np.exp(-d * d / (2 * sig * sig)), 0.0)
            cell = j * 6 + i
            assert W[cell] == pytest.approx(w.sum(), rel=1e-9, abs=1e-300)
            for c in range(C):
                if w.sum() > 0:
                    assert out[c, cell] == pytest.approx((w * v[c]).sum() / w.sum(), rel=1e-9)
                else:
                    assert np.isnan(out[c, cell])
    # channel subset and cell subset select the same numbers
    o2, W2, _ = oracle.grid(lon, lat, v, m, fwhm, channels=[2, 0], cells=[7, 29, 0])
    np.testing.assert_array_equal(o2, out[[2, 0]][:, [7, 29, 0]])
    np.testing.assert_array_equal(W2, W[[7, 29, 0]])


# ---------------------------------------------------------------- invariants
def test_linearity_and_lon_translation():
    """grid(a v1 + b v2) = a grid(v1) + b grid(v2) (shared weights);
    shifting every lon and the map reference by the same amount leaves values unchanged."""
    rng = np.random.default_rng(5)
    N = 4000
    lon = 30 + rng.uniform(-0.15, 0.15, N)
    lat = 41 + rng.uniform(-0.15, 0.15, N)
    v1 = rng.normal(10, 1, N)
    v2 = rng.normal(3, 1, N)
    m = mk_map(16, 16, 30.0, 41.0, 1.0 / 60)
    fwhm = 3.0 / 60
    vals = np.stack([v1, v2, 2.0 * v1 - 3.0 * v2]).astype(np.float32)
    out, W, _ = oracle.grid(lon, lat, vals, m, fwhm)
    a = vals.astype(np.float64)
    ok = W > 0
    lhs = out[2, ok]
    rhs = (2.0 * out[0, ok] - 3.0 * out[1, ok])
    # vals[2] was rounded to fp32, so compare against its exact fp64 combination
    err_in = np.abs(a[2] - (2 * a[0] - 3 * a[1])).max()
    np.testing.assert_allclose(lhs, rhs, atol=1e-10 + 4 * err_in)
    m2 = dict(m, crval_lon=m["crval_lon"] + 100.0)
    out2, W2, _ = oracle.grid(lon + 100.0, lat, vals, m2, fwhm)
    np.testing.assert_allclose(W2, W, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(out2[:, ok], out[:, ok], rtol=1e-10)


def test_field_straddling_lon_zero():
    """Reading R9: a map centred on lon 0 sees samples at lon 359.9x as neighbours."""
    rng = np.random.default_rng(9)
    lon = (rng.uniform(-0.1, 0.1, 2000) + 360.0) % 360.0
    lat = rng.uniform(-0.1, 0.1, 2000)
    m = mk_map(12, 12, 0.0, 0.0, 1.0 / 60)
    _, W, cnt = oracle.grid(lon, lat, None, m, 3.0 / 60)
    _, Wr, cntr = oracle.grid(np.where(lon > 180, lon - 360, lon), lat, None, m, 3.0 / 60)
    assert np.all(cnt > 0)
    np.testing.assert_array_equal(cnt, cntr)
    np.testing.assert_allclose(W, Wr, rtol=1e-9)


def test_neighbour_sets_match_sklearn_balltree():
    """Independent library: sklearn BallTree(metric='haversine').query_radius must give the
    oracle's neighbour sets exactly (Algorithm 1's d <= R set), barring ties within 1e-12 of R."""
    from sklearn.neighbors import BallTree
    rng = np.random.default_rng(21)
    N = 20000
    lon = 30 + rng.uniform(-0.3, 0.3, N)
    lat = 41 + rng.uniform(-0.3, 0.3, N)
    m = mk_map(30, 30, 30.0, 41.0, 1.0 / 60)
    fwhm = 3.0 / 60
    off, idx = oracle.neighbours(lon, lat, m, fwhm)
    R = 3.0 * math.radians(fwhm / FWHM2SIG)
    tree = BallTree(np.radians(np.stack([lat, lon], 1)), metric="haversine")
    jj, ii = np.divmod(np.arange(900), 30)
    cl = 30 + (ii + 1 - 15.5) / 60
    cb = 41 + (jj + 1 - 15.5) / 60
    res = tree.query_radius(np.radians(np.stack([cb, cl], 1)), r=R)
    ties = 0
    for q in range(900):
        a = set(idx[off[q]:off[q + 1]].tolist())
        b = set(res[q].tolist())
        for s in a ^ b:
            d = dist_atan2(cl[q], cb[q], lon[s], lat[s])
            assert abs(d - R) <= 1e-12 * R, (q, s, d, R)
            ties += 1
    assert ties == 0
    assert off[-1] > 900 * 50
    # CSR lists are ascending original index
    for q in range(0, 900, 37):
        seg = idx[off[q]:off[q + 1]]
        assert np.all(np.diff(seg) > 0)


def test_thread_count_does_not_change_results():
    rng = np.random.default_rng(2)
    lon = 30 + rng.uniform(-0.1, 0.1, 3000)
    lat = 41 + rng.uniform(-0.1, 0.1, 3000)
    v = rng.normal(5, 1, (2, 3000)).astype(np.float32)
    m = mk_map(10, 10, 30.0, 41.0, 1.0 / 60)
    a = oracle.grid(lon, lat, v, m, 3.0 / 60, nthreads=1)
    b = oracle.grid(lon, lat, v, m, 3.0 / 60, nthreads=4)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_tophat_kernel_is_plain_neighbour_mean():
    """SPEC.md:117-126 tophat kernel (1 for d <= R, else 0): W is the neighbour count and the
    map is the plain mean of the values within R.  Neighbour sets from sklearn's BallTree
    (haversine) and the mean from numpy: nothing shared with the oracle's loop."""
    from sklearn.neighbors import BallTree
    rng = np.random.default_rng(33)
    N = 6000
    lon = 30 + rng.uniform(-0.2, 0.2, N)
    lat = 41 + rng.uniform(-0.2, 0.2, N)
    v = rng.normal(10, 2, (2, N)).astype(np.float32)
    m = mk_map(16, 14, 30.0, 41.0, 1.0 / 60)
    fwhm = 3.0 / 60
    out, W, cnt = oracle.grid(lon, lat, v, m, fwhm, kernel="tophat")
    R = 3.0 * math.radians(fwhm / FWHM2SIG)
    tree = BallTree(np.radians(np.stack([lat, lon], 1)), metric="haversine")
    jj, ii = np.divmod(np.arange(16 * 14), 16)
    cl = 30 + (ii + 1 - 8.5) / 60
    cb = 41 + (jj + 1 - 7.5) / 60
    res = tree.query_radius(np.radians(np.stack([cb, cl], 1)), r=R)
    for q in range(16 * 14):
        s = res[q]
        assert W[q] == len(s) == cnt[q]
        if len(s):
            np.testing.assert_allclose(out[:, q], v[:, s].astype(np.float64).mean(1), rtol=1e-12)
        else:
            assert np.all(np.isnan(out[:, q]))
    # the Gaussian and the tophat share the support: identical neighbour counts and blanks
    og, Wg, cg = oracle.grid(lon, lat, v, m, fwhm)
    np.testing.assert_array_equal(cg, cnt)
    assert np.all((Wg > 0) == (W > 0))


# ------------------------------------------------------------------ NEXT-4 variants (readings R24, R25)
def test_integer_sample_weights_equal_duplicated_samples():
    """Per-sample weights multiply the kernel weight (R25): an integer weight k gives exactly
    what k copies of the sample give (0 removes it) -- a pin by construction, not by formula."""
    rng = np.random.default_rng(25)
    n = 300
    lon = 30 + (rng.random(n) - 0.5) * 0.2
    lat = 41 + (rng.random(n) - 0.5) * 0.2
    vals = (10 + rng.standard_normal((2, n))).astype(np.float32)
    wgt = rng.integers(0, 4, n)
    m = {"nx": 9, "ny": 8, "crval_lon": 30.0, "crval_lat": 41.0, "crpix_x": 5.0, "crpix_y": 4.5,
         "cdelt_lon": 0.02, "cdelt_lat": 0.02}
    o, W, _ = oracle.grid(lon, lat, vals, m, 0.05, sample_weights=wgt.astype(np.float64))
    rep = np.repeat(np.arange(n), wgt)
    o2, W2, _ = oracle.grid(lon[rep], lat[rep], vals[:, rep], m, 0.05)
    np.testing.assert_allclose(W, W2, rtol=1e-13, atol=0)
    np.testing.assert_array_equal(np.isnan(o), np.isnan(o2))
    ok = ~np.isnan(o)
    np.testing.assert_allclose(o[ok], o2[ok], rtol=1e-12)


def test_mask_equals_removing_the_masked_sample_from_its_channel():
    """Masking (R24): a non-finite value leaves both sums of its channel -- channel c's map
    equals the map gridded without the masked samples of c; the weight map keeps them."""
    rng = np.random.default_rng(24)
    n = 400
    lon = 30 + (rng.random(n) - 0.5) * 0.2
    lat = 41 + (rng.random(n) - 0.5) * 0.2
    vals = (10 + rng.standard_normal((3, n))).astype(np.float32)
    vals[0, rng.choice(n, 40, replace=False)] = np.nan
    vals[2, rng.choice(n, 15, replace=False)] = np.inf
    m = {"nx": 9, "ny": 8, "crval_lon": 30.0, "crval_lat": 41.0, "crpix_x": 5.0, "crpix_y": 4.5,
         "cdelt_lon": 0.02, "cdelt_lat": 0.02}
    o, W, _ = oracle.grid(lon, lat, vals, m, 0.05, mask=True)
    _, Wp, _ = oracle.grid(lon, lat, vals, m, 0.05)
    np.testing.assert_array_equal(W, Wp)
    for c in range(3):
        keep = np.isfinite(vals[c])
        oc, _, _ = oracle.grid(lon[keep], lat[keep], vals[c:c + 1, keep], m, 0.05)
        np.testing.assert_array_equal(np.isnan(o[c]), np.isnan(oc[0]))
        ok = ~np.isnan(oc[0])
        np.testing.assert_allclose(o[c][ok], oc[0][ok], rtol=1e-13)
    # propagate (R15): a NaN makes every cell within R NaN
    op, _, _ = oracle.grid(lon, lat, vals, m, 0.05)
    assert np.isnan(op[0]).sum() > np.isnan(o[0]).sum()


@pytest.mark.parametrize("proj", ["tan", "sin"])
def test_zenithal_projection_cell_centres(proj):
    """Reading R26: gnomonic (TAN) / orthographic (SIN) cell centres.  Closed forms with the
    reference point at (0, 0): along the x axis lon = atan(x) (TAN) or asin(x) (SIN) with
    lat = 0, along the y axis lat = atan(y) / asin(y); anywhere, the great-circle distance from
    the reference point is atan(r) / asin(r) (r = the offset in radians); the reference
    pixel is the reference point."""
    f = math.atan if proj == "tan" else math.asin
    m = {"nx": 21, "ny": 21, "crval_lon": 0.0, "crval_lat": 0.0, "crpix_x": 11.0, "crpix_y": 11.0,
         "cdelt_lon": 1.5, "cdelt_lat": 1.5, "projection": proj}
    for i in range(21):
        x = (i + 1 - 11.0) * 1.5
        lon, lat = oracle.cell_centre(m, i, 10)
        assert abs(lon - math.degrees(f(math.radians(x)))) < 1e-12 and abs(lat) < 1e-12
        lon, lat = oracle.cell_centre(m, 10, i)
        assert abs(lat - math.degrees(f(math.radians(x)))) < 1e-12 and abs(lon) < 1e-12
    m2 = dict(m, crval_lon=30.0, crval_lat=41.0, cdelt_lon=-0.7, cdelt_lat=0.4)
    c0 = oracle.cell_centre(m2, 10, 10)
    assert abs(c0[0] - 30.0) < 1e-12 and abs(c0[1] - 41.0) < 1e-12
    for i, j in [(0, 0), (3, 17), (20, 5), (12, 9)]:
        x, y = (i + 1 - 11.0) * -0.7, (j + 1 - 11.0) * 0.4
        r = math.radians(math.hypot(x, y))
        lon, lat = oracle.cell_centre(m2, i, j)
        d = oracle.distance_deg(30.0, 41.0, lon, lat)
        assert abs(d - math.degrees(f(r))) < 1e-10, (i, j, d)
        # east (x > 0 with cdelt_lon < 0 means i left of crpix) -> the sign of the lon offset
        assert (lon - 30.0) * x > 0 or abs(x) < 1e-12
