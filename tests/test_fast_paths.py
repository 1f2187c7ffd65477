"""Exactness of the integer fast paths the fusion kernels use in place of a
division (rf_volume.cu). The device code computes the same expressions; the
GPU parity tests check the resulting voxels bit for bit."""
import numpy as np


def test_colour_average_magic_multiply_is_exact():
    """colour_avg (rf_volume.cu): lround((c w + in) / (w + 1)) = (2n + d) / (2d) with
    n = c w + in and d = w + 1, computed as the high word of the 32-bit product
    (2n + d) * ceil(2^32 / 2d) (one IMAD.HI). Every numerator < 2^17 and every d in
    1..256 is checked (tools/micro/colour_magic.c runs the same check over the
    (c, w, in) triples the update can see)."""
    num = np.arange(0, 1 << 17, dtype=np.uint64)
    for d in range(1, 257):
        m = ((1 << 32) + 2 * d - 1) // (2 * d)
        assert m < (1 << 32)
        np.testing.assert_array_equal((num * np.uint64(m)) >> np.uint64(32), num // np.uint64(2 * d))


def test_colour_average_matches_rounded_quotient():
    """(2n + d) / (2d) is lround(n / d) (ties away from zero) for the value ranges used."""
    c = np.arange(256, dtype=np.int64)[:, None, None]
    w = np.arange(256, dtype=np.int64)[None, :, None]
    x = np.array([0, 1, 127, 128, 254, 255], dtype=np.int64)[None, None, :]
    n = c * w + x
    d = w + 1
    want = np.floor(n / d + 0.5).astype(np.int64)  # n, d >= 0: lround = floor(q + 1/2)
    np.testing.assert_array_equal((2 * n + d) // (2 * d), want)


def _fma(x, y, z):
    """fma(x, y, z) with one rounding (Fraction arithmetic is exact; float() of a
    Fraction rounds to nearest even)."""
    from fractions import Fraction
    return float(Fraction(x) * Fraction(y) + Fraction(z))


def test_walk_division_by_reciprocal_is_correctly_rounded():
    """div_rn (rf_volume.cu, the ray-segment setup of WalkGridSegment,
    tsdf_volume.hpp:149-185): q = RN(a rb), r = fma(-q, b, a), q' = fma(r, rb, q) with
    rb = RN(1/b) equals the IEEE quotient a / b. Checked on the walk's operand ranges:
    pixel offsets over focal lengths, and world coordinates over brick extents
    (8 voxel sizes; the reciprocal there is RN(1/s) scaled by 2^-3)."""
    rng = np.random.default_rng(7)
    cases = []
    for f in (525.0, 517.3, 481.2, 600.0, 910.7, 1000.0 / 3.0):
        for u in rng.uniform(-700.0, 700.0, 300):
            cases.append((float(u), f, 1.0 / f))
        for u in range(-64, 65):
            cases.append((float(u) + 0.5, f, 1.0 / f))
    for s in (0.005, 0.01, 0.02, 0.0075, 0.004):
        ext, rext = 8.0 * s, (1.0 / s) * (1.0 / 8.0)
        assert rext == 1.0 / ext
        for w in rng.uniform(-20.0, 20.0, 600):
            cases.append((float(w), ext, rext))
        for k in range(-50, 51):  # coordinates on and next to brick faces
            for w in (k * ext, np.nextafter(k * ext, np.inf), np.nextafter(k * ext, -np.inf)):
                cases.append((float(w), ext, rext))
    for a, b, rb in cases:
        q = a * rb
        r = _fma(-q, b, a)
        assert _fma(r, rb, q) == a / b or (a == 0.0), (a, b)


def test_running_average_f32_fast_path_agrees_with_division():
    """div_f32 (rf_volume.cu): f32((sdf w + u) / (w + k)) from q = RN(a * RN(1/b));
    when every f64 within 2^-50 relative of q rounds to the same f32 (lo == hi),
    that f32 is the f32 of the correctly rounded quotient. Checked on 2e6 random
    updates over the ranges the carve and integrate updates see (numpy float64 is
    IEEE binary64 without contraction, like the kernels under -fmad=false)."""
    rng = np.random.default_rng(11)
    n = 2_000_000
    tau = 0.1
    sdf = rng.uniform(-tau, tau, n).astype(np.float32).astype(np.float64)
    w = rng.integers(0, 65, n).astype(np.float64)
    k = np.where(rng.random(n) < 0.5, 1.0, rng.integers(1, 5, n).astype(np.float64))
    u = np.where(rng.random(n) < 0.8, rng.uniform(-tau, tau, n), tau * k)
    a = sdf * w + u
    b = w + k
    rb = 1.0 / b
    q = a * rb
    lo = (q * (1.0 - 2.0 ** -50)).astype(np.float32)
    hi = (q * (1.0 + 2.0 ** -50)).astype(np.float32)
    fast = lo == hi
    assert fast.mean() > 0.99
    np.testing.assert_array_equal(lo[fast], (a[fast] / b[fast]).astype(np.float32))


def test_projection_rounding_fast_path_agrees_with_lround():
    """project_lround (rf_volume.cu): away from half-integers (margin 1e-9) the
    pixel from num * rz + c, rz within an ulp of 1/z (the kernel's branch-free
    reciprocal; perturbed by +-1 ulp here), rounds like lround(num / z + c)
    (Project, geometry.hpp:46-48). 2e6 random camera points in and around a
    1280x720 view, plus points forced onto exact half-integers, which the
    margin sends to the exact path."""
    rng = np.random.default_rng(5)
    n = 2_000_000
    z = rng.uniform(1e-3, 6.0, n)
    f = rng.choice([50.0, 525.0, 1050.0], n)
    c = rng.choice([31.5, 319.5, 639.5], n)
    x = rng.uniform(-0.5, 1.5, n) * 1280.0
    X = (x - c) * z / f
    X[: n // 10] = (np.round(x[: n // 10]) + 0.5 - c[: n // 10]) * z[: n // 10] / f[: n // 10]  # ties
    num = f * X
    rz = 1.0 / z
    ulp = rng.integers(-1, 2, n)
    rz = np.where(ulp > 0, np.nextafter(rz, np.inf), np.where(ulp < 0, np.nextafter(rz, 0.0), rz))
    xa = num * rz + c
    fr = xa - np.floor(xa)
    fast = (np.abs(xa) < 1e6) & (np.abs(fr - 0.5) > 1e-9)
    v = num / z + c
    lround = np.where(v >= 0, np.floor(v + 0.5), np.ceil(v - 0.5))
    assert fast.mean() > 0.85 and (~fast).sum() > 0
    np.testing.assert_array_equal(np.rint(xa[fast]), lround[fast])
