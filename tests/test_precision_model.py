"""Error model of the tensor-core engine's products ("Tolerance budget"),
emulated in numpy: no GPU, no oracle.

Per (sample, cell) pair the engine forms v*w as
    v_hi * w_hi                                  (kind::tf32 MMA: 11-bit x 11-bit, exact in fp32)
  + bf16(v) * bf16(w_lo) + bf16(v_lo) * bf16(w_hi)   (one kind::f16 MMA, K = 16 element pairs)
with x_hi = x rounded to tf32 on the bit pattern (tc::split_tf32) and x_lo = x - x_hi (exact in
fp32), bf16 conversions rounding to nearest even (cvt.rn.bf16x2.f32).  The claims checked here:
|x_lo| <= 2^-11 |x| and bf16 rounds to <= 2^-8 relative, so each correction term is off by
<= 2 * 2^-11 * 2^-8 = 2^-18 of v*w and a product by <= 2^-17 (worst case; unbiased, RMS
~2^-20.6), and the normalised sums (Eq. 1) stay far inside north_star's 1e-5 bar.
"""
import numpy as np


def tf32_split(x):
    x = np.asarray(x, np.float32)
    hi = ((x.view(np.uint32) + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
    lo = (x - hi).astype(np.float32)
    return hi, lo


def bf16(x):
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16              # round to nearest even
    return (r << 16).astype(np.uint32).view(np.float32)


def mixed_product(v, w):
    vh, vl = tf32_split(v)
    wh, wl = tf32_split(w)
    f = np.float64
    return (f(vh) * f(wh)) + f(bf16(v)) * f(bf16(wl)) + f(bf16(vl)) * f(bf16(wh))


def test_split_is_exact_and_hi_is_tf32():
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(100_000) * 10.0 ** rng.uniform(-6, 6, 100_000)).astype(np.float32)
    hi, lo = tf32_split(x)
    assert np.all(hi.astype(np.float64) + lo.astype(np.float64) == x.astype(np.float64))
    assert np.all((hi.view(np.uint32) & 0x1FFF) == 0)
    assert np.all(np.abs(lo) <= np.abs(x) * 2.0 ** -11 * (1 + 1e-6))


def test_hi_product_is_exact_in_fp32():
    rng = np.random.default_rng(2)
    vh, _ = tf32_split(rng.uniform(-100, 100, 100_000).astype(np.float32))
    wh, _ = tf32_split(rng.uniform(0.0111, 1.0, 100_000).astype(np.float32))
    exact = vh.astype(np.float64) * wh.astype(np.float64)
    assert np.all((vh * wh).astype(np.float64) == exact)   # 11 + 11 significant bits fit in 24


def test_product_error_bound():
    rng = np.random.default_rng(3)
    n = 200_000
    v = (rng.standard_normal(n) * 10.0 ** rng.uniform(-4, 4, n)).astype(np.float32)
    # Gaussian weights on [0, R] with R = 3 sigma, and the tophat's w = 1
    d = rng.uniform(0, 3, n)
    w = np.exp(-0.5 * d * d).astype(np.float32)
    w[: n // 10] = 1.0
    exact = v.astype(np.float64) * w.astype(np.float64)
    err = (mixed_product(v, w) - exact) / np.abs(exact)
    rel = np.abs(err)
    assert rel.max() < 2.0 ** -17
    assert np.sqrt(np.mean(err ** 2)) < 2.0 ** -20      # typical error
    assert abs(err.mean()) < 2.0 ** -26                  # round to nearest: no bias
    # the tophat (w_lo = 0): only bf16(v_lo) is rounded, <= 2^-11 * 2^-8 = 2^-19
    assert rel[: n // 10].max() < 2.0 ** -19


def test_weighted_mean_far_inside_tolerance():
    """Eq. 1 over ~700 neighbours with zero-mean and offset values: the normalised sum from the
    mixed products (summed in fp64 here, i.e. without the accumulator's own rounding, which
    DESIGN.md bounds separately) stays below 1e-6 relative to the scale of the values."""
    rng = np.random.default_rng(4)
    worst = 0.0
    for trial in range(200):
        k = 700
        d = rng.uniform(0, 3, k)
        w = np.exp(-0.5 * d * d).astype(np.float32)
        v = (rng.standard_normal(k) * 3.0 + (10.0 if trial % 2 else 0.0)).astype(np.float32)
        S = mixed_product(v, w).sum()
        Se = (v.astype(np.float64) * w.astype(np.float64)).sum()
        W = w.astype(np.float64).sum()
        scale = np.abs(v).max()
        worst = max(worst, abs(S / W - Se / W) / scale)
    assert worst < 1e-6
