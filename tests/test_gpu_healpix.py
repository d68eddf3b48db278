"""The HEALPix-indexed plan (NEXT-2): the paper's own LUT (Fig. 4/5) and
Algorithm 1's ring-by-ring gather, on the GPU, for the fields the lon/lat
bin index does not serve (polar caps, >= 180 degrees of longitude, R > 1 degree).

* ang2pix_ring (the plan's key, computed on the device) against the ring-scheme layout
  (SPEC.md:17-110 examples), the pixel-centre round trip, and HEALPix's defining property
  (equal-area pixels: uniform directions fill every pixel alike, a chi-square bound);
* gridded maps against the fp64 oracle (values, W and blank pattern), and the gather's
  neighbour sets against the oracle's d <= R sets, exactly.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2207_04584_b200 import HegridError, Plan, hegrid_healpix_ang2pix
from parity_util import compare

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ the pixelisation
def _ring_layout(nside):
    """(start, len, z, f) of rings 1 .. 4 nside - 1 from the published ring-scheme layout."""
    rows = []
    start = 0
    for i in range(1, 4 * nside):
        if i < nside:
            n, z, f = 4 * i, 1 - i * i / (3 * nside * nside), 0.5
        elif i <= 3 * nside:
            n, z, f = 4 * nside, 4 / 3 - 2 * i / (3 * nside), (0.0 if (i + nside) % 2 else 0.5)
        else:
            ii = 4 * nside - i
            n, z, f = 4 * ii, -1 + ii * ii / (3 * nside * nside), 0.5
        rows.append((start, n, z, f))
        start += n
    assert start == 12 * nside * nside
    return rows


@pytest.mark.parametrize("nside", [1, 2, 4, 8, 64])
def test_ang2pix_pixel_centre_round_trip(nside):
    th, ph, want = [], [], []
    for start, n, z, f in _ring_layout(nside):
        for j in range(n):
            th.append(math.acos(z))
            ph.append((j + f) * 2 * math.pi / n)
            want.append(start + j)
    got = hegrid_healpix_ang2pix(nside, np.array(th), np.array(ph))
    np.testing.assert_array_equal(got, np.array(want))


def test_ang2pix_spec_examples():
    """nside=1 equator -> ring 2 (pixels 4..7); nside=2 pixel 0 sits
    on cap ring 1 at z = 11/12; longitude is taken modulo 2 pi."""
    p = hegrid_healpix_ang2pix(1, np.array([math.pi / 2]), np.array([0.0]))[0]
    assert 4 <= p <= 7
    z = 11 / 12
    assert hegrid_healpix_ang2pix(2, np.array([math.acos(z)]), np.array([math.pi / 4]))[0] == 0
    a = hegrid_healpix_ang2pix(8, np.array([1.0, 1.0]), np.array([2.0, 2.0 + 6 * math.pi]))
    assert a[0] == a[1]
    with pytest.raises(HegridError):
        hegrid_healpix_ang2pix(3, np.array([1.0]), np.array([1.0]))
    with pytest.raises(HegridError):
        hegrid_healpix_ang2pix(4, np.array([4.0]), np.array([1.0]))


@pytest.mark.parametrize("nside", [4, 16])
def test_pixels_have_equal_area(nside):
    """Uniform directions on the sphere fill the 12 nside^2 pixels equally (HEALPix is an
    equal-area pixelisation): every count within 6 sigma of the mean, chi-square plausible."""
    rng = np.random.default_rng(nside)
    n = 3_000_000
    z = rng.uniform(-1, 1, n)
    ph = rng.uniform(0, 2 * math.pi, n)
    pix = hegrid_healpix_ang2pix(nside, np.arccos(z), ph)
    npix = 12 * nside * nside
    cnt = np.bincount(pix, minlength=npix)
    assert cnt.shape[0] == npix and pix.min() >= 0
    mean = n / npix
    assert np.all(np.abs(cnt - mean) <= 6 * math.sqrt(mean)), (cnt.min(), cnt.max(), mean)
    chi2 = float(((cnt - mean) ** 2 / mean).sum())
    assert chi2 < npix + 6 * math.sqrt(2 * npix), chi2


# ------------------------------------------------------------------ gridding through the LUT
def _polar_field(seed=88, n=20000):
    rng = np.random.default_rng(seed)
    # uniform on the cap lat >= 84.5 (area-uniform: z uniform)
    z = rng.uniform(math.sin(math.radians(84.5)), 1.0, n)
    lat = np.degrees(np.arcsin(z))
    lon = rng.uniform(0, 360, n)
    m = {"nx": 24, "ny": 12, "crval_lon": 180.0, "crval_lat": 87.0, "crpix_x": 12.5, "crpix_y": 6.5,
         "cdelt_lon": 15.0, "cdelt_lat": 0.45}
    return lon, lat, m, 0.6          # kernel FWHM 0.6 deg: R = 0.76 deg


def _sky_field(seed=7, n=60000):
    rng = np.random.default_rng(seed)
    z = rng.uniform(-1, 1, n)
    lat = np.degrees(np.arcsin(z))
    lon = rng.uniform(-180, 180, n)
    m = {"nx": 36, "ny": 17, "crval_lon": 0.0, "crval_lat": 0.0, "crpix_x": 18.5, "crpix_y": 9.0,
         "cdelt_lon": 10.0, "cdelt_lat": 10.0}
    return lon, lat, m, 4.0          # R = 5.1 deg


def _values(n, C, seed=3):
    rng = np.random.default_rng(seed)
    return (10.0 + rng.standard_normal((C, n))).astype(np.float32)


@pytest.mark.parametrize("field", ["polar", "sky"])
@pytest.mark.parametrize("kernel", ["gaussian", "tophat"])
def test_healpix_plan_parity(field, kernel):
    lon, lat, m, fwhm = _polar_field() if field == "polar" else _sky_field()
    vals = _values(lon.shape[0], 3)
    with Plan(lon, lat, m, fwhm, kernel=kernel) as p:
        info = p.info()
        assert info["index"] == 2 and info["nside"] >= 1    # AUTO chose HEALPix
        out, W = p.grid(vals)
        off, idx = p.neighbours()
    o, Wo, _ = oracle.grid(lon, lat, vals, m, fwhm, 3.0, kernel=kernel)
    st = compare(out, W, o, Wo)
    assert st["covered"] > 0
    ooff, oidx = oracle.neighbours(lon, lat, m, fwhm, 3.0)     # the d <= R set (any kernel)
    np.testing.assert_array_equal(off, ooff)
    np.testing.assert_array_equal(idx, oidx)
    if kernel == "tophat":       # W is the neighbour count
        np.testing.assert_array_equal(W.reshape(-1), np.diff(off).astype(np.float32))


def test_bin_index_refuses_polar_field_healpix_serves_it():
    lon, lat, m, fwhm = _polar_field(n=2000)
    with pytest.raises(HegridError):
        Plan(lon, lat, m, fwhm, index="bins")
    with Plan(lon, lat, m, fwhm, index="healpix") as p:
        assert p.info()["index"] == 2


def test_healpix_forced_on_an_ordinary_field_matches_oracle():
    """The HEALPix LUT on the cfg1 geometry (where AUTO takes the bins): same maps and the
    same neighbour sets as the oracle."""
    import synth
    w = synth.CONFIGS["cfg1"]
    lon, lat = synth.coords(w)
    vals = synth.values(w, lon, lat).numpy()
    lon, lat = lon.numpy(), lat.numpy()
    with Plan(lon, lat, w.map, w.fwhm_deg, index="healpix") as p:
        assert p.info()["index"] == 2
        out, W = p.grid(vals)
        off, idx = p.neighbours()
    with Plan(lon, lat, w.map, w.fwhm_deg) as q:
        assert q.info()["index"] == 1
    o, Wo, _ = oracle.grid(lon, lat, vals, w.map, w.fwhm_deg, w.support)
    compare(out, W, o, Wo)
    ooff, oidx = oracle.neighbours(lon, lat, w.map, w.fwhm_deg, w.support)
    np.testing.assert_array_equal(off, ooff)
    np.testing.assert_array_equal(idx, oidx)


def test_healpix_device_path_and_empty():
    import torch
    lon, lat, m, fwhm = _sky_field(n=5000)
    vals = _values(lon.shape[0], 5)
    with Plan(lon, lat, m, fwhm) as p:
        out_h, W_h = p.grid(vals)
        out_d, W_d = p.grid(torch.as_tensor(vals).cuda())
        assert np.array_equal(np.asarray(out_h).view(np.uint32), out_d.cpu().numpy().view(np.uint32))
    with Plan(np.zeros(0), np.zeros(0), m, fwhm, index="healpix") as p:
        out, W = p.grid(np.zeros((2, 0), np.float32))
        assert np.all(np.isnan(out)) and np.all(np.asarray(W) == 0)
