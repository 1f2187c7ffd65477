"""Trajectory evaluation of the product (rf_ate_rmse / rf_rpe_over_time: host
C++ in the CUDA library, no device work) against the reference's KATs and the
oracle. The product aligns with Horn's quaternion method, the oracle with the
reference's SVD route (evaluation.cpp:41-50): agreement to 1e-12 checks both."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import eval_kats

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1905_02082_b200",
                   "librefusion_b200.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="CUDA library not built")


@pytest.fixture(scope="module")
def G():
    from paper_1905_02082_b200 import api
    return api


@pytest.mark.parametrize("kat", [eval_kats.kat_ate_rigid_invariance, eval_kats.kat_ate_radial_inflation,
                                 eval_kats.kat_ate_association, eval_kats.kat_rpe_drift],
                         ids=lambda f: f.__name__)
def test_product_trajectory_kat(G, kat):
    kat(G)


def noisy_pair(seed, n=300, planar=False):
    """Ground truth orbit and an estimate = rigid offset * (gt + drift noise),
    sampled at jittered timestamps (some pairs fail to associate)."""
    rng = np.random.default_rng(seed)
    gt, est = [], []
    offset = eval_kats.small_pose(rng.normal(size=3), rng.normal(size=3), rng.uniform(-2, 2))
    for i in range(n):
        a = 0.02 * i
        t = [np.cos(a) * 2, 0.0 if planar else 0.3 * np.sin(3 * a), np.sin(a) * 2]
        p = eval_kats.small_pose(t, [0, 1, 0], a)
        gt.append((i / 30.0, p))
        q = p.copy()
        q[9:] += rng.normal(scale=0.01, size=3)
        est.append((i / 30.0 + rng.uniform(-0.03, 0.03), eval_kats.compose(offset, q)))
    return est, gt


@pytest.mark.parametrize("seed,planar", [(1, False), (2, True), (3, False)])
def test_ate_rpe_match_oracle(G, seed, planar):
    est, gt = noisy_pair(seed, planar=planar)
    r_g, al_g, n_g = G.ate_rmse(est, gt)
    r_o, al_o, n_o = O.ate_rmse(est, gt)
    assert n_g == n_o and 3 <= n_g < len(gt)
    assert abs(r_g - r_o) <= 1e-12 * max(1.0, r_o)
    np.testing.assert_allclose(al_g, al_o, rtol=0, atol=1e-9)
    for delta in (0.5, 1.0, 3.0):
        ts_g, e_g = G.rpe_over_time(est, gt, delta)
        ts_o, e_o = O.rpe_over_time(est, gt, delta)
        np.testing.assert_array_equal(ts_g, ts_o)
        np.testing.assert_allclose(e_g, e_o, rtol=0, atol=1e-12)
