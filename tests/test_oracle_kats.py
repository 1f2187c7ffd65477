"""Pins the CPU oracle to the reference's own known-answer tests.

Each test restates one reference test case (file:line under
/root/reference/proj/tests) against the oracle restatement. The reference
cannot be built here (Eigen3/libpng/doctest absent), so these KATs are what
anchors the oracle to the reference's behaviour.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests import helpers as H


def vcfg(**kw):
    return O.vol_cfg(voxel_size=0.02, truncation=0.1, **kw)


def flat_frame(depth, k, gray=128.0):
    d = np.full((k.height, k.width), depth, dtype=np.float32)
    rgb = np.full((k.height, k.width, 3), int(gray), dtype=np.uint8)
    return d, rgb


# --------------------------------------------------------------- spatial hash
def np_hash(c):
    c = np.asarray(c, dtype=np.int64).reshape(-1, 3)
    u = (c & 0xFFFFFFFF).astype(np.uint64)
    return (u[:, 0] * np.uint64(73856093)) ^ (u[:, 1] * np.uint64(19349669)) ^ (u[:, 2] * np.uint64(83492791))


def test_hash_insert_find_against_dict():  # test_spatial_hash.cpp:20-50
    rng = np.random.default_rng(4242)
    coords = rng.integers(-4000, 4001, size=(200000, 3)).astype(np.int32)
    m = O.HashMap()
    vals, inserted = m.insert(coords, np.arange(200000, dtype=np.uint32))
    ref = {}
    for i, c in enumerate(map(tuple, coords)):
        fresh = c not in ref
        if fresh:
            ref[c] = i
        assert inserted[i] == fresh
        assert vals[i] == ref[c]
    assert m.size() == len(ref)
    keys = np.array(list(ref.keys()), dtype=np.int32)
    v, found = m.find(keys)
    assert found.all()
    assert (v == np.array(list(ref.values()))).all()
    absent = rng.integers(5000, 9001, size=(10000, 3))
    assert not m.find(absent)[1].any()


def test_hash_growth_and_duplicates():  # test_spatial_hash.cpp:72-95
    m = O.HashMap(16)
    n = 3000
    c = np.stack([np.arange(n), -np.arange(n), 7 * np.arange(n)], 1)
    m.insert(c, np.arange(n, dtype=np.uint32))
    assert m.size() == n
    cap = m.capacity()
    assert cap >= n * 4 // 3 and (cap & (cap - 1)) == 0
    v, f = m.find(c)
    assert f.all() and (v == np.arange(n)).all()
    m2 = O.HashMap()
    assert m2.insert([[1, 2, 3]], [10])[1][0]
    val, ins = m2.insert([[1, 2, 3]], [99])
    assert not ins[0] and val[0] == 10 and m2.size() == 1


def test_hash_function_matches_numpy_and_spreads():  # test_spatial_hash.cpp:97-125
    rng = np.random.default_rng(1)
    sample = rng.integers(-(1 << 20), 1 << 20, size=(50, 3))
    for c, h in zip(sample, np_hash(sample)):
        assert O.hash_coord(*c) == int(h)
    x, y, z = np.meshgrid(np.arange(-128, 128), np.arange(-128, 128), np.arange(64), indexing="ij")
    h = np_hash(np.stack([x.ravel(), y.ravel(), z.ravel()], 1))
    counts = np.bincount((h & np.uint64(255)).astype(np.int64), minlength=256)
    exp = counts.sum() / 256
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 < 2000 and counts.max() < 1.5 * exp and counts.min() > 0.5 * exp


def test_hash_million_keys():  # acceptance.cpp:539-579 (criterion 7)
    rng = np.random.default_rng(123)
    keys = np.unique(rng.integers(-(1 << 20), 1 << 20, size=(1050000, 3)), axis=0)[:1000000]
    keys = keys[rng.permutation(len(keys))]
    m = O.HashMap()
    _, ins = m.insert(keys, np.arange(len(keys), dtype=np.uint32))
    assert ins.all()
    v, f = m.find(keys)
    assert f.all() and (v == np.arange(len(keys))).all()
    probes = rng.integers(-(1 << 20), 1 << 20, size=(1000000, 3))
    keyset = set(map(tuple, keys[:200000].tolist()))
    _, f2 = m.find(probes)
    # A false hit would need the random probe to be an inserted key.
    hits = probes[f2]
    assert len(hits) < 5


# --------------------------------------------------------------- volume
def test_flat_frame_projective_distance():  # test_tsdf.cpp:49-83
    vol = O.Volume(vcfg())
    k = O.small_intrinsics()
    d, rgb = flat_frame(0.5, k)
    vol.allocate_for_frame(d, k, O.IDENTITY)
    vol.integrate(d, rgb, k, O.IDENTITY)
    band = clamped = untouched = 0
    for vz in range(5, 40):
        vox, found = vol.get_voxels([[0, 0, vz]])
        if not found[0]:
            continue
        z = (vz + 0.5) * 0.02
        exp = 0.5 - z
        if exp < -0.1:
            assert vox["weight"][0] == 0
            untouched += 1
        elif exp > 0.1:
            assert vox["weight"][0] == 1
            assert vox["sdf"][0] == pytest.approx(0.1)
            assert vox["r"][0] == 0
            clamped += 1
        else:
            assert vox["weight"][0] == 1
            assert vox["sdf"][0] == pytest.approx(exp, rel=1e-6, abs=1e-7)
            assert vox["r"][0] == 128
            band += 1
    assert band >= 9 and clamped >= 1 and untouched >= 1


def test_weights_saturate():  # test_tsdf.cpp:85-97
    vol = O.Volume(vcfg())
    k = O.small_intrinsics()
    d, rgb = flat_frame(0.5, k)
    vol.allocate_for_frame(d, k, O.IDENTITY)
    for _ in range(80):
        vol.integrate(d, rgb, k, O.IDENTITY)
    vox, found = vol.get_voxels([[0, 0, 24]])
    assert found[0] and vox["weight"][0] == 64
    assert vox["sdf"][0] == pytest.approx(0.01, rel=1e-5)


def test_color_running_mean():  # test_tsdf.cpp:99-121
    vol = O.Volume(vcfg())
    k = O.small_intrinsics()
    d, _ = flat_frame(0.5, k)
    bright = np.zeros((k.height, k.width, 3), np.uint8)
    bright[:] = (200, 100, 40)
    dark = np.zeros_like(bright)
    dark[:] = (100, 50, 20)
    vol.allocate_for_frame(d, k, O.IDENTITY)
    vol.integrate(d, bright, k, O.IDENTITY)
    vol.integrate(d, dark, k, O.IDENTITY)
    vox, _ = vol.get_voxels([[0, 0, 24]])
    assert vox["weight"][0] == 2
    assert (vox["r"][0], vox["g"][0], vox["b"][0]) == (150, 75, 30)


def test_masked_integration_and_allocation():  # test_tsdf.cpp:123-158
    k = O.small_intrinsics()
    d, rgb = flat_frame(0.5, k)
    mask = np.zeros((k.height, k.width), np.uint8)
    mask[:, : k.width // 2] = 1

    def bp(u, v, z):
        return np.array([(u - k.cx) / k.fx * z, (v - k.cy) / k.fy * z, z])

    left, right = bp(k.width / 4.0, k.height / 2.0, 0.5), bp(3.0 * k.width / 4.0, k.height / 2.0, 0.5)
    vox_of = lambda p: np.floor(p / 0.02).astype(np.int32)
    vol = O.Volume(vcfg())
    vol.allocate_for_frame(d, k, O.IDENTITY)
    vol.integrate(d, rgb, k, O.IDENTITY, mask)
    vm, fm = vol.get_voxels([vox_of(left)])
    vo, fo = vol.get_voxels([vox_of(right)])
    assert fm[0] and fo[0] and vm["weight"][0] == 0 and vo["weight"][0] == 1
    vol2 = O.Volume(vcfg())
    vol2.allocate_for_frame(d, k, O.IDENTITY, mask)
    ext = 0.16
    lb = np.floor(left / ext).astype(int)
    coords, _ = vol2.export(with_voxels=False)
    assert not any((coords == lb).all(1))


def _wavy_volume(cfg):
    vol = O.Volume(cfg)
    H.fill_volume(vol, (-0.4, -0.4, 0.0), (0.4, 0.4, 0.8), H.wavy_probe, H.wavy_probe_intensity)
    return vol


def test_trilinear_matches_eight_corner_sum():  # test_tsdf.cpp:160-200
    vol = _wavy_volume(vcfg())
    rng = np.random.default_rng(5)
    pts = np.stack([rng.uniform(-0.3, 0.3, 500), rng.uniform(-0.3, 0.3, 500), rng.uniform(0.1, 0.7, 500)], 1)
    val, _, valid = vol.sample(pts, 0)
    ival, _, ivalid = vol.sample(pts, 1)
    assert valid.all() and ivalid.all()
    s = 0.02
    for p, v, iv in zip(pts, val, ival):
        g = p / s - 0.5
        base = np.floor(g).astype(int)
        f = g - base
        exp = expi = 0.0
        for dz in range(2):
            for dy in range(2):
                for dx in range(2):
                    c, _ = vol.get_voxels([base + [dx, dy, dz]])
                    w = (f[0] if dx else 1 - f[0]) * (f[1] if dy else 1 - f[1]) * (f[2] if dz else 1 - f[2])
                    exp += w * float(c["sdf"][0])
                    expi += w * (0.2126 * c["r"][0] + 0.7152 * c["g"][0] + 0.0722 * c["b"][0])
        assert v == pytest.approx(exp, rel=1e-12, abs=1e-15)
        assert iv == pytest.approx(expi, rel=1e-9)


def test_gradient_differentiates_interpolant():  # test_tsdf.cpp:202-223
    vol = O.Volume(vcfg())
    H.fill_volume(vol, (-0.4, -0.4, 0.0), (0.4, 0.4, 0.8), H.wavy_probe)
    rng = np.random.default_rng(6)
    pts = np.stack([rng.uniform(-0.25, 0.25, 200), rng.uniform(-0.25, 0.25, 200), rng.uniform(0.15, 0.65, 200)], 1)
    v, g, ok = vol.sample(pts, 2)
    v0, _, _ = vol.sample(pts, 0)
    assert ok.all()
    np.testing.assert_allclose(v, v0, rtol=1e-12, atol=1e-15)
    h = 1e-7
    for axis in range(3):
        dp = np.zeros(3)
        dp[axis] = h
        fd = (vol.sample(pts + dp, 0)[0] - vol.sample(pts - dp, 0)[0]) / (2 * h)
        np.testing.assert_allclose(g[:, axis], fd, rtol=1e-4, atol=1e-6)


def test_central_difference_ramp():  # test_tsdf.cpp:225-237
    vol = O.Volume(vcfg())
    H.fill_volume(vol, (-0.4, -0.4, 0.0), (0.4, 0.4, 0.8), lambda p: 0.3 * p[0] - 0.2 * p[1] + 0.1 * p[2])
    _, g, ok = vol.sample([[0.05, -0.03, 0.4]], 4)
    assert ok[0]
    np.testing.assert_allclose(g[0], [0.3, -0.2, 0.1], rtol=1e-5)
    assert not vol.sample([[0.39, 0.0, 0.4]], 4)[2][0]


def test_segment_walk_covers_dense_sampling():  # test_tsdf.cpp:239-256
    rng = np.random.default_rng(11)
    cell = 0.16
    for _ in range(200):
        a, b = rng.uniform(-0.9, 0.9, 3), rng.uniform(-0.9, 0.9, 3)
        walked = set(map(tuple, O.walk_segment(a, b, cell).tolist()))
        length = np.linalg.norm(b - a)
        steps = max(2, int(length / (cell * 1e-3)))
        t = np.arange(steps + 1) / steps
        pts = a[None] + (b - a)[None] * t[:, None]
        sampled = set(map(tuple, np.floor(pts / cell).astype(int).tolist()))
        assert sampled <= walked
        assert len(walked) <= len(sampled) + 3


def test_allocation_covers_band():  # test_tsdf.cpp:258-282
    vol = O.Volume(vcfg())
    k = O.small_intrinsics()
    d, _ = H.make_frame(k, lambda u, v: 0.45 + 0.1 * math.sin(0.3 * u) * math.cos(0.4 * v))
    vol.allocate_for_frame(d, k, O.IDENTITY)
    coords, _ = vol.export(with_voxels=False)
    have = set(map(tuple, coords.tolist()))
    rng = np.random.default_rng(3)
    for _ in range(300):
        u, v = int(rng.integers(0, k.width)), int(rng.integers(0, k.height))
        z = float(d[v, u])
        p = np.array([(u - k.cx) / k.fx * z, (v - k.cy) / k.fy * z, z])
        dirn = p / np.linalg.norm(p)
        for off in (-0.099, -0.05, 0.0, 0.05, 0.099):
            q = p + dirn * off
            assert tuple(np.floor(q / 0.16).astype(int).tolist()) in have


def test_carve_closed_form():  # test_tsdf.cpp:284-311
    vol = O.Volume(vcfg())
    k = O.small_intrinsics()
    d, rgb = flat_frame(0.5, k)
    vol.allocate_for_frame(d, k, O.IDENTITY)
    for _ in range(3):
        vol.integrate(d, rgb, k, O.IDENTITY)
    vox, _ = vol.get_voxels([[0, 0, 24]])
    s0 = float(vox["sdf"][0])
    assert vox["weight"][0] == 3
    far, _ = flat_frame(1.5, k)
    for n in range(1, 31):
        vol.carve(far, k, O.IDENTITY)
        vox, _ = vol.get_voxels([[0, 0, 24]])
        assert float(vox["sdf"][0]) == pytest.approx((3 * s0 + n * 0.1) / (3 + n), rel=1e-5)
    assert vox["sdf"][0] > 0.05
    nb = vol.num_blocks()
    vol.carve(far, k, O.IDENTITY)
    assert vol.num_blocks() == nb


def test_carve_leaves_band_alone():  # test_tsdf.cpp:313-324
    vol = O.Volume(vcfg())
    k = O.small_intrinsics()
    d, rgb = flat_frame(0.5, k)
    vol.allocate_for_frame(d, k, O.IDENTITY)
    vol.integrate(d, rgb, k, O.IDENTITY)
    before, _ = vol.get_voxels([[0, 0, 24]])
    vol.carve(d, k, O.IDENTITY)
    after, _ = vol.get_voxels([[0, 0, 24]])
    assert before["sdf"][0] == after["sdf"][0]


def test_block_budget():  # test_tsdf.cpp:372-382
    vol = O.Volume(vcfg(max_blocks=4))
    for x in range(4):
        assert vol.allocate_block((x, 0, 0))
    with pytest.raises(O.ResourceLimit):
        vol.allocate_block((4, 0, 0))
    assert not vol.allocate_block((0, 0, 0))


def test_integration_thread_invariance():  # test_tsdf.cpp:384-406
    k = O.small_intrinsics()
    d, rgb = H.make_frame(k, lambda u, v: 0.4 + 0.003 * u + 0.002 * v, lambda u, v: (u * 3 + v * 5) % 256)
    out = []
    for threads in (1, 4):
        vol = O.Volume(vcfg())
        vol.allocate_for_frame(d, k, O.IDENTITY)
        vol.integrate(d, rgb, k, O.IDENTITY, None, threads)
        vol.carve(d, k, O.IDENTITY, threads)
        out.append(vol.export())
    assert (out[0][0] == out[1][0]).all()
    assert out[0][1].tobytes() == out[1][1].tobytes()


# --------------------------------------------------------------- registration
def wavy_sdf(p):
    return 0.06 * math.sin(3.0 * p[0] + 0.7) * math.cos(2.0 * p[1] - 0.4) + 0.04 * math.sin(2.2 * p[2])


def wavy_intensity(p):
    return 120.0 + 70.0 * math.sin(1.7 * p[0] - 0.3) * math.cos(1.3 * p[2] + 0.2)


def wavy_volume(voxel=0.025, lo=(-0.6, -0.5, 0.05), hi=(0.6, 0.5, 0.95)):
    vol = O.Volume(O.vol_cfg(voxel_size=voxel, truncation=0.1))
    H.fill_volume(vol, lo, hi, wavy_sdf, wavy_intensity)
    return vol


def wavy_frame():
    k = O.small_intrinsics()
    d, rgb = H.make_frame(k, lambda u, v: 0.45 + 0.04 * math.sin(0.4 * u) * math.cos(0.3 * v),
                          lambda u, v: 110.0 + 60.0 * math.sin(0.25 * u + 0.1 * v))
    return k, d, rgb


def test_pyramid_rules():  # test_registration.cpp:50-77
    k = O.small_intrinsics(8, 4, 10.0)
    d, rgb = H.make_frame(k, lambda u, v: 1.0 + u + 8.0 * v, lambda u, v: 10.0 * u + v)
    d[1, 2] = 0.0
    mask = np.zeros((4, 8), np.uint8)
    mask[2, 5] = 1
    pyr = O.build_pyramid(d, rgb, k, 3, mask)
    assert pyr[1]["depth"].shape == (2, 4) and pyr[2]["depth"].shape == (1, 2)
    assert pyr[1]["intr"][0] == pytest.approx(5.0)
    assert pyr[1]["depth"][0, 0] == pytest.approx(1.0)
    assert pyr[1]["depth"][0, 1] == pytest.approx(3.0)
    assert pyr[1]["intensity"][0, 0] == pytest.approx((0 + 10 + 1 + 11) / 4.0, rel=1e-6)
    assert pyr[1]["mask"][1, 2] == 1 and pyr[1]["mask"][0, 0] == 0 and pyr[2]["mask"][0, 1] == 1


def test_gradient_matches_finite_differences():  # test_registration.cpp:79-118
    vol = wavy_volume()
    k, d, rgb = wavy_frame()
    rng = np.random.default_rng(17)
    checked = 0
    h = 1e-5
    for _ in range(20):
        t = rng.uniform(-0.02, 0.02, 3)
        axis = rng.uniform(-1, 1, 3)
        if np.linalg.norm(axis) < 1e-3:
            axis = np.array([0, 0, 1.0])
        pose = H.small_pose(t, axis, rng.uniform(-0.017, 0.017))
        at = vol.linearize(d, rgb, k, pose)
        assert at["valid"] > 500
        for i in range(6):
            step = np.zeros(6)
            step[i] = h
            plus = vol.linearize(d, rgb, k, H.compose(O.expmap(step), pose))
            minus = vol.linearize(d, rgb, k, H.compose(O.expmap(-step), pose))
            assert plus["valid"] == at["valid"] == minus["valid"]
            fd = (plus["error"] - minus["error"]) / (2 * h)
            an = 2.0 * at["b"][i]
            assert abs(fd - an) / max(abs(fd), abs(an), 1e-6) < 1e-3
            checked += 1
    assert checked == 120


def plane_volume():
    vol = O.Volume(O.vol_cfg(voxel_size=0.02, truncation=0.1))
    H.fill_volume(vol, (-1.0, -1.0, 0.3), (1.0, 1.0, 0.7), lambda p: p[2] - 0.5)
    return vol


def test_plane_shift_residuals():  # test_registration.cpp:120-140
    vol = plane_volume()
    k = O.small_intrinsics()
    d = np.full((k.height, k.width), 0.5, np.float32)
    err, sq, valid = vol.evaluate_depth_error(d, k, H.small_pose((0, 0, 0.01), (0, 0, 1), 0.0))
    assert valid.all()
    np.testing.assert_allclose(sq, 1e-4, rtol=1e-3)
    assert err == pytest.approx(1e-4 * valid.sum(), rel=1e-3)


def test_plane_is_degenerate():  # test_registration.cpp:142-151
    vol = plane_volume()
    k = O.small_intrinsics()
    d = np.full((k.height, k.width), 0.5, np.float32)
    assert vol.linearize(d, None, k, O.IDENTITY, O.reg_cfg(color_weight=0.0))["degenerate"]


class Corner:
    """test_registration.cpp:157-180"""

    def __init__(self):
        from paper_1905_02082_b200 import scenes
        self.scene = O.Scene(scenes.corner_scene())
        self.k = self.scene.k
        self.r = self.scene.render(0)
        self.view = self.scene.camera(0)[1]
        self.vol = O.Volume(O.vol_cfg(voxel_size=0.02, truncation=0.1))
        self.vol.allocate_for_frame(self.r["depth"], self.k, self.view)
        self.vol.integrate(self.r["depth"], self.r["rgb"], self.k, self.view)

    def perturbed(self):
        return H.compose(self.view, H.small_pose((0.03, -0.02, 0.04), (1.0, 1.0, 0.0), 3.0 * math.pi / 180))

    def error_of(self, pose):
        return H.compose(H.inverse(self.view), pose)


@pytest.fixture(scope="module")
def corner():
    return Corner()


@pytest.mark.parametrize("cw", [0.0, 0.025])
def test_registration_recovers_perturbation(corner, cw):  # test_registration.cpp:184-204
    r = corner.vol.register(corner.r["depth"], corner.r["rgb"], corner.k, corner.perturbed(), None,
                            O.reg_cfg(color_weight=cw))
    e = corner.error_of(r["pose"])
    assert np.linalg.norm(e[9:]) < 5e-3
    assert H.rotation_angle(e) < 0.5 * math.pi / 180
    if cw > 0:
        assert r["valid_residuals"] > 1000


def test_lm_never_increases_error():  # test_registration.cpp:206-218
    vol = wavy_volume(0.04, (-1.6, -1.4, 0.05), (1.6, 1.4, 1.2))
    k, d, rgb = wavy_frame()
    init = H.small_pose((0.02, 0.01, -0.02), (0.0, 1.0, 0.3), 1.5 * math.pi / 180)
    at = vol.linearize(d, rgb, k, init)
    r = vol.register(d, rgb, k, init)
    assert r["final_error"] <= at["error"] * (1 + 1e-12)


def test_masked_pixels_do_not_influence(corner):  # test_registration.cpp:220-262
    k = corner.k
    clean = corner.r["depth"]
    corrupted = clean.copy()
    mask = np.zeros((k.height, k.width), np.uint8)
    sl = (slice(None), slice(0, k.width // 3))
    valid = corrupted[sl] > 0
    corrupted[sl] = np.where(valid, corrupted[sl] + np.float32(0.05), corrupted[sl])
    mask[sl] = 1
    a = corner.vol.register(clean, corner.r["rgb"], k, corner.perturbed(), mask)
    b = corner.vol.register(corrupted, corner.r["rgb"], k, corner.perturbed(), mask)
    c = corner.vol.register(corrupted, corner.r["rgb"], k, corner.perturbed(), None)
    diff = H.compose(H.inverse(a["pose"]), b["pose"])
    assert np.linalg.norm(diff[9:]) < 1e-12 and H.rotation_angle(diff) < 1e-7
    assert np.linalg.norm(corner.error_of(c["pose"])[9:]) > 0.02
    assert np.linalg.norm(corner.error_of(a["pose"])[9:]) < 0.1
    assert b["res_valid"][sl].sum() > 0


def test_tracking_lost():  # test_registration.cpp:264-271
    vol = O.Volume(O.vol_cfg(voxel_size=0.025, truncation=0.1))
    H.fill_volume(vol, (-0.2, -0.2, 0.4), (0.2, 0.2, 0.6), wavy_sdf)
    k = O.small_intrinsics()
    d = np.full((k.height, k.width), 3.0, np.float32)
    with pytest.raises(O.TrackingLost):
        vol.register(d, None, k, O.IDENTITY)


def test_expmap_logmap_roundtrip():  # test_geometry.cpp:37-79
    rng = np.random.default_rng(9)
    for _ in range(50):
        xi = np.concatenate([rng.uniform(-1, 1, 3), rng.uniform(-1.5, 1.5, 3)])
        np.testing.assert_allclose(O.logmap(O.expmap(xi)), xi, atol=1e-9)
    xi = np.array([0.1, -0.2, 0.3, 1e-8, -2e-8, 3e-8])
    p = O.expmap(xi)
    R = p[:9].reshape(3, 3)
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-12)
    # closed form against the matrix exponential of the se(3) generator
    from scipy.linalg import expm
    xi = np.array([0.3, -0.1, 0.2, 0.4, -0.7, 0.2])
    G = np.zeros((4, 4))
    w = xi[3:]
    G[:3, :3] = [[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]]
    G[:3, 3] = xi[:3]
    np.testing.assert_allclose(O.pose_matrix(O.expmap(xi)), expm(G), atol=1e-12)


def test_ldlt_matches_numpy():
    rng = np.random.default_rng(0)
    for _ in range(100):
        A = rng.normal(size=(6, 6))
        A = A @ A.T + 1e-3 * np.eye(6)
        b = rng.normal(size=6)
        x, ok = O.ldlt6(A, b)
        assert ok
        np.testing.assert_allclose(A @ x, b, rtol=1e-8, atol=1e-8)


# --------------------------------------------------------------- dynamics mask
def test_threshold_strict():  # test_mask.cpp:31-45
    sq = np.array([[0.005, 0.0051, 1.0, 0.0049]], np.float32)
    valid = np.array([[1, 1, 0, 1]], np.uint8)
    assert O.threshold(sq, valid).tolist() == [[0, 1, 0, 0]]


def test_erode_dilate():  # test_mask.cpp:47-106
    m = np.zeros((9, 9), np.uint8)
    m[2:7, 2:7] = 1
    e = O.erode(m, 1)
    assert e.sum() == 9 and e[4, 4] and e[3, 3] and not e[2, 2]
    dl = O.dilate(e, 1)
    assert (dl <= m).all() and dl.sum() == 25
    full = np.ones((5, 5), np.uint8)
    e2 = O.erode(full, 2)
    assert e2.sum() == 1 and e2[2, 2] == 1 and O.dilate(e2, 2).sum() == 25
    rng = np.random.default_rng(1)
    r = (rng.integers(0, 2, (5, 7))).astype(np.uint8)
    assert (O.erode(r, 0) == r).all() and (O.dilate(r, 0) == r).all()
    a = (rng.integers(0, 4, (9, 12)) == 0).astype(np.uint8)
    b = np.maximum(a, (rng.integers(0, 5, (9, 12)) == 0).astype(np.uint8))
    assert (O.dilate(a, 2) <= O.dilate(b, 2)).all()


def step_depth():
    d = np.zeros((5, 5), np.float32)
    d[:, :3] = 1.0
    d[:, 3:] = 1.5
    return d


def test_floodfill_hand_trace_and_seed_invariance():  # test_mask.cpp:112-156, acceptance.cpp:494-529
    d = step_depth()
    seeds = np.zeros((5, 5), np.uint8)
    seeds[1, 1] = 1
    g = O.floodfill(seeds, d, 0.007, 4)
    exp = np.zeros((5, 5), np.uint8)
    exp[:, :3] = 1
    assert (g == exp).all()
    near = [(x, y) for y in range(5) for x in range(3)]
    rng = np.random.default_rng(77)
    for _ in range(100):
        rng.shuffle(near)
        s = np.zeros((5, 5), np.uint8)
        for x, y in near[: 1 + int(rng.integers(0, 4))]:
            s[y, x] = 1
        assert (O.floodfill(s, d, 0.007, 4) == exp).all()


def test_floodfill_invalid_depth_and_asymmetric_rule():  # test_mask.cpp:158-192
    d = np.ones((1, 4), np.float32)
    d[0, 2] = 0
    s = np.zeros((1, 4), np.uint8)
    s[0, 0] = 1
    assert O.floodfill(s, d, 0.05).tolist() == [[1, 1, 0, 0]]
    s = np.zeros((1, 4), np.uint8)
    s[0, 2] = 1
    assert O.floodfill(s, d, 0.05).tolist() == [[0, 0, 1, 0]]
    d = np.array([[2.0, 2.012, 2.03]], np.float32)
    s = np.array([[1, 0, 0]], np.uint8)
    assert O.floodfill(s, d, 0.007).tolist() == [[1, 1, 0]]


def test_floodfill_connectivity():  # test_mask.cpp:194-205
    d = np.ones((2, 2), np.float32)
    d[0, 1] = 2.0
    d[1, 0] = 2.0
    s = np.array([[1, 0], [0, 0]], np.uint8)
    assert O.floodfill(s, d, 0.007, 4)[1, 1] == 0
    assert O.floodfill(s, d, 0.007, 8)[1, 1] == 1


def test_build_mask_composition():  # test_mask.cpp:207-241
    n = 16
    d = np.full((n, n), 2.0, np.float32)
    sq = np.full((n, n), 0.0001, np.float32)
    d[4:10, 4:10] = 1.0
    sq[4:10, 4:10] = 0.009
    sq[14, 14] = 0.009
    m = O.build_mask(sq, np.ones((n, n), np.uint8), d, O.mask_cfg(erode_radius=1, dilate_radius=1))
    assert m[4:10, 4:10].all()
    assert m[14, 14] == 0 and m[0, 0] == 0 and m[4, 3] == 1 and m[4, 10] == 1 and m[4, 2] == 0


# --------------------------------------------------------------- raycast
def test_raycast_plane():  # test_refine.cpp:242-265 (ray-march half of RenderVirtualDepth)
    k = O.small_intrinsics()
    vol = O.Volume(vcfg())
    d, rgb = flat_frame(0.5, k)
    for _ in range(4):
        vol.allocate_for_frame(d, k, O.IDENTITY)
        vol.integrate(d, rgb, k, O.IDENTITY)
    out = vol.raycast(O.IDENTITY, k)
    inner = out[4:-4, 4:-4]
    assert (inner > 0).all()
    np.testing.assert_allclose(inner, 0.5, rtol=2e-3)


# --------------------------------------------------------------- mesh
def test_sphere_mesh():  # test_mesh.cpp:43-126
    center, radius = np.array([0.1, -0.05, 0.4]), 0.25
    vol = O.Volume(vcfg())
    m = radius + 0.1
    H.fill_volume(vol, center - m, center + m, lambda p: float(np.linalg.norm(p - center) - radius))
    v, c, f = vol.extract_mesh(1)
    assert len(v) > 1000 and len(f) > 1000
    r = np.linalg.norm(v.astype(np.float64) - center, axis=1)
    assert np.abs(r - radius).max() < 0.25 * 0.02
    a, b, cc = (v[f[:, i]].astype(np.float64) for i in range(3))
    n = np.cross(b - a, cc - a)
    centroid = (a + b + cc) / 3
    assert (np.sum(n * (centroid - center), 1) > 0).mean() > 0.99
    edges = {}
    for tri in f:
        for i in range(3):
            e = tuple(sorted((int(tri[i]), int(tri[(i + 1) % 3]))))
            edges[e] = edges.get(e, 0) + 1
    assert all(cnt == 2 for cnt in edges.values())
    v1, c1, f1 = vol.extract_mesh(1, threads=4)
    assert (v1 == v).all() and (f1 == f).all()
