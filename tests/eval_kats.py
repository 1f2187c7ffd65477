"""The reference's evaluation known-answer tests (proj/tests/test_eval.cpp and
acceptance.cpp:594-620), restated against an implementation object `E` that
exposes ate_rmse / rpe_over_time / nearest_distances / distance_cdf (the
oracle on CPU, the product on the GPU). Random draws use numpy instead of
std::mt19937: the checks are properties, not vectors."""
import numpy as np
import pytest


def small_pose(t, axis, angle):
    """SmallPose (test_util.hpp:100-103): AngleAxis(angle, axis) + t, as 12 doubles."""
    a = np.asarray(axis, np.float64)
    a = a / np.linalg.norm(a)
    k = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    r = np.eye(3) + np.sin(angle) * k + (1 - np.cos(angle)) * (k @ k)
    return np.concatenate([r.reshape(9), np.asarray(t, np.float64)])


def compose(a, b):
    ra, rb = a[:9].reshape(3, 3), b[:9].reshape(3, 3)
    return np.concatenate([(ra @ rb).reshape(9), ra @ b[9:] + a[9:]])


def inverse(a):
    rt = a[:9].reshape(3, 3).T
    return np.concatenate([rt.reshape(9), -(rt @ a[9:])])


def random_trajectory(rng, count):
    """RandomTrajectory (test_eval.cpp:18-28)."""
    out = []
    for i in range(count):
        t = 2.0 * rng.uniform(-1, 1, 3)
        axis = rng.uniform(-1, 1, 3)
        out.append((0.1 * i, small_pose(t, axis, rng.uniform(-1, 1))))
    return out


def kat_ate_rigid_invariance(E):  # test_eval.cpp:32-47
    rng = np.random.default_rng(42)
    gt = random_trajectory(rng, 25)
    offset = small_pose([1.5, -0.7, 2.2], [0.3, 0.8, -0.5], 0.9)
    est = [(t, compose(offset, p)) for t, p in gt]
    rmse, al, pairs = E.ate_rmse(est, gt)
    assert pairs == len(gt)
    assert rmse < 1e-9
    exp = inverse(offset)
    assert np.linalg.norm(al[:9] - exp[:9]) < 1e-9
    assert np.linalg.norm(al[9:] - exp[9:]) < 1e-9


def kat_ate_radial_inflation(E):  # test_eval.cpp:49-68
    eps = 0.01
    pts = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    gt = [(float(i), np.concatenate([np.eye(3).reshape(9), p])) for i, p in enumerate(pts)]
    est = [(float(i), np.concatenate([np.eye(3).reshape(9), (1 + eps) * np.asarray(p, float)])) for i, p in
           enumerate(pts)]
    rmse, al, pairs = E.ate_rmse(est, gt)
    assert pairs == 6
    assert rmse == pytest.approx(eps, rel=1e-9)
    assert np.linalg.norm(al[:9] - np.eye(3).reshape(9)) < 1e-9
    assert np.linalg.norm(al[9:]) < 1e-9


def kat_ate_association(E):  # test_eval.cpp:70-88
    rng = np.random.default_rng(3)
    gt = random_trajectory(rng, 20)
    est = [(gt[i][0] + 0.003, gt[i][1]) for i in range(0, len(gt), 2)]
    rmse, _, pairs = E.ate_rmse(est, gt, 0.02)
    assert pairs == len(est)
    assert rmse < 1e-9
    with pytest.raises(RuntimeError):
        E.ate_rmse(gt[:2], gt)
    shifted = [(t + 100.0, p) for t, p in gt]
    with pytest.raises(RuntimeError):
        E.ate_rmse(shifted, gt)


def kat_rpe_drift(E):  # test_eval.cpp:90-113
    gt, est = [], []
    for k in range(91):
        t = k / 30.0
        gt.append((t, np.concatenate([np.eye(3).reshape(9), [0.1 * t, 0, 0]])))
        est.append((t, np.concatenate([np.eye(3).reshape(9), [0.105 * t, 0, 0]])))
    ts, err = E.rpe_over_time(est, gt, 1.0, 0.02)
    assert len(err) == 61
    assert np.allclose(err, 0.005, rtol=1e-9, atol=0)
    assert ts[0] == pytest.approx(0.0) and ts[-1] == pytest.approx(2.0)
    _, zero = E.rpe_over_time(gt, gt, 1.0, 0.02)
    assert len(zero) > 0 and np.all(zero < 1e-12)
    assert len(E.rpe_over_time(est, gt, 10.0, 0.02)[1]) == 0
    with pytest.raises(ValueError):
        E.rpe_over_time(est, gt, 0.0, 0.02)


def brute_force(q, r):
    """min over the reference of ||(p - q).cast<double>()|| with the oracle's
    summation order (x^2 + y^2) + z^2."""
    q = np.asarray(q, np.float32)
    r = np.asarray(r, np.float32)
    out = np.empty(len(q))
    for i in range(len(q)):
        d = (r - q[i]).astype(np.float64)  # f32 difference, then widened
        out[i] = np.sqrt(np.min((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]))
    return out


def kat_nearest_brute_force(E):  # test_eval.cpp:115-144
    rng = np.random.default_rng(11)
    uni = lambda n: rng.uniform(-1.0, 2.0, (n, 3)).astype(np.float32)  # noqa: E731
    ref = np.concatenate([uni(600), 50.0 + uni(20)]).astype(np.float32)
    qs = np.concatenate([uni(300), (30.0 * uni(30)).astype(np.float32), ref[5:6]]).astype(np.float32)
    got = E.nearest_distances(qs, ref)
    assert len(got) == len(qs)
    np.testing.assert_array_equal(got, brute_force(qs, ref))
    assert got[-1] == 0.0
    assert len(E.nearest_distances(np.zeros((0, 3), np.float32), ref)) == 0
    with pytest.raises(ValueError):
        E.nearest_distances(qs, np.zeros((0, 3), np.float32))


def kat_nearest_acceptance(E):  # acceptance.cpp:600-616
    rng = np.random.default_rng(5)
    qs = rng.uniform(-2, 2, (1000, 3)).astype(np.float32)
    ref = rng.uniform(-2, 2, (1000, 3)).astype(np.float32)
    np.testing.assert_array_equal(E.nearest_distances(qs, ref), brute_force(qs, ref))


def kat_distance_cdf(E):  # test_eval.cpp:146-172
    edges = [0.0025, 0.005, 0.01, 0.05]
    cdf = E.distance_cdf([0.001, 0.003, 0.007, 0.02], edges)
    assert list(cdf) == [25.0, 50.0, 75.0, 100.0]
    assert E.distance_cdf([0.005], edges)[1] == 100.0  # on an edge counts as inside
    rng = np.random.default_rng(8)
    rd = rng.uniform(0.0, 0.1, 500)
    wide = [0.006 * i for i in range(1, 21)]
    rc = E.distance_cdf(rd, wide)
    assert np.all(np.diff(rc) >= 0)
    assert rc[-1] == pytest.approx(100.0)
    with pytest.raises(ValueError):
        E.distance_cdf([], edges)
    with pytest.raises(ValueError):
        E.distance_cdf([0.001, 0.003], [0.01, 0.005])


ALL = [kat_ate_rigid_invariance, kat_ate_radial_inflation, kat_ate_association, kat_rpe_drift,
       kat_nearest_brute_force, kat_nearest_acceptance, kat_distance_cdf]
