"""Exactness of the integer fast paths the fusion kernels use in place of a
division (rf_volume.cu). The device code computes the same expressions; the
GPU parity tests check the resulting voxels bit for bit."""
import numpy as np


def test_colour_average_magic_multiply_is_exact():
    """colour_avg: lround((c w + in) / (w + 1)) = (2n + d) / (2d) with n = c w + in and
    d = w + 1, computed as ((2n + d) * ceil(2^40 / 2d)) >> 40. Every numerator
    < 2^17 and every d in 1..256 is checked."""
    num = np.arange(0, 1 << 17, dtype=np.uint64)
    for d in range(1, 257):
        m = np.uint64(((1 << 40) + 2 * d - 1) // (2 * d))
        np.testing.assert_array_equal((num * m) >> np.uint64(40), num // np.uint64(2 * d))


def test_colour_average_matches_rounded_quotient():
    """(2n + d) / (2d) is lround(n / d) (ties away from zero) for the value ranges used."""
    c = np.arange(256, dtype=np.int64)[:, None, None]
    w = np.arange(256, dtype=np.int64)[None, :, None]
    x = np.array([0, 1, 127, 128, 254, 255], dtype=np.int64)[None, None, :]
    n = c * w + x
    d = w + 1
    want = np.floor(n / d + 0.5).astype(np.int64)  # n, d >= 0: lround = floor(q + 1/2)
    np.testing.assert_array_equal((2 * n + d) // (2 * d), want)
