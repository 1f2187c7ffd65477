"""Parity of the CUDA path (through the C ABI) against the CPU oracle on
identical inputs.

Bars:
  * allocation: identical brick key set and identical occupied-slot bitmap of
    the hash at the GPU's capacity — bit-exact;
  * integrate / carve voxels: bit-exact (sdf f32, weight, rgb);
  * sampling, residual images, raycast depth, masks: bit-exact;
  * normal equations: relative error <= 1e-9 (fp64 reduction order differs);
  * poses: <= 1e-4 m and <= 1e-4 rad (BASELINE.json north_star).
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests import helpers as H

pytestmark = pytest.mark.gpu

POSE_TOL_T = 1e-4
POSE_TOL_R = 1e-4


# ------------------------------------------------------------------ helpers
def gk(k):  # oracle intrinsics -> C ABI intrinsics
    return G.intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_scale)


def gcfg(o: O.OVolCfg):
    return G.volume_config(voxel_size=o.voxel_size, truncation=o.truncation, block_side=o.block_side,
                           max_weight=o.max_weight, carve_weight=o.carve_weight, min_depth=o.min_depth,
                           max_depth=o.max_depth, carve_clip=o.carve_clip, max_blocks=o.max_blocks)


def greg(o: O.ORegCfg):
    return G.registration_config(color_weight=o.color_weight, pyramid_levels=o.pyramid_levels,
                                 max_iterations=o.max_iterations, lm_lambda_init=o.lm_lambda_init,
                                 lm_lambda_up=o.lm_lambda_up, lm_lambda_down=o.lm_lambda_down,
                                 convergence_eps=o.convergence_eps, min_valid_residuals=o.min_valid_residuals)


def pair(ocfg):
    return O.Volume(ocfg), G.TsdfVolume(gcfg(ocfg))


def frame(k, depth, rgb=None, t=0.0):
    return G.Frame(depth=depth, rgb=rgb, intrinsics=gk(k), timestamp=t)


def canonical(coords, vox):
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    return coords[order], (None if vox is None else vox[order])


def assert_volumes_identical(ov, gv, check_occupancy=True):
    oc, ovox = canonical(*ov.export())
    gc, gvox = canonical(*gv.export())
    assert oc.shape == gc.shape, f"block count {len(oc)} vs {len(gc)}"
    assert (oc == gc).all(), "block key sets differ"
    assert ovox.tobytes() == gvox.tobytes(), "voxels differ"
    if check_occupancy:
        cap = gv.hash_capacity()
        assert (ov.hash_occupancy(cap) == gv.hash_occupancy()).all(), "hash occupancy differs"


def pose_error(a, b):
    d = H.compose(H.inverse(a), b)
    return float(np.linalg.norm(d[9:])), H.rotation_angle(d)


def wavy_frame(k, seed):
    rng = np.random.default_rng(seed)
    a, b, c = rng.uniform(0.3, 0.6), rng.uniform(0.05, 0.15), rng.uniform(0.1, 0.5)
    d, rgb = H.make_frame(k, lambda u, v: a + b * math.sin(c * u) * math.cos(0.37 * v),
                          lambda u, v: 127 + 120 * math.sin(0.3 * u + 0.2 * v + seed))
    d[rng.random(d.shape) < 0.05] = 0.0  # dropouts
    return d, rgb


# ------------------------------------------------------------------ volume
def test_flat_frame_allocate_integrate_bitexact():
    k = O.small_intrinsics()
    ov, gv = pair(O.vol_cfg(voxel_size=0.02))
    d = np.full((k.height, k.width), 0.5, np.float32)
    rgb = np.full((k.height, k.width, 3), 128, np.uint8)
    ov.allocate_for_frame(d, k, O.IDENTITY)
    ov.integrate(d, rgb, k, O.IDENTITY)
    gv.allocate_for_frame(frame(k, d, rgb), O.IDENTITY)
    gv.integrate(frame(k, d, rgb), O.IDENTITY)
    assert_volumes_identical(ov, gv)


@pytest.mark.parametrize("voxel", [0.01, 0.02])
def test_lockstep_carve_allocate_integrate_bitexact(voxel):
    k = O.small_intrinsics(64, 48, 50.0)
    ov, gv = pair(O.vol_cfg(voxel_size=voxel))
    rng = np.random.default_rng(7)
    for i in range(6):
        d, rgb = wavy_frame(k, i)
        pose = H.small_pose(rng.uniform(-0.05, 0.05, 3), rng.uniform(-1, 1, 3), rng.uniform(-0.1, 0.1))
        mask = (rng.random(d.shape) < 0.1).astype(np.uint8) if i % 2 else None
        ov.carve(d, k, pose)
        gv.carve(frame(k, d), pose)
        ov.allocate_for_frame(d, k, pose, mask)
        gv.allocate_for_frame(frame(k, d), pose, mask)
        ov.integrate(d, rgb, k, pose, mask)
        gv.integrate(frame(k, d, rgb), pose, mask)
        assert_volumes_identical(ov, gv)


@pytest.mark.parametrize("shift", [0.01, 0.03, -0.05])
def test_projection_ties_take_the_exact_path(shift):
    """Voxels whose projection lands on a pixel boundary (x = fx X / Z + cx at a
    half-integer, where lround's tie rule decides): with f s = 1, cx = 31.5 and the
    camera shifted by half a voxel, every voxel of the z = 0.25 m layer projects
    to within an ulp of a half-integer. k_fuse's reciprocal fast path must hand
    those to the exact division (rf_volume.cu project_lround), so the voxels stay
    bit-identical to the oracle's."""
    k = O.small_intrinsics(64, 48, 50.0)  # cx = 31.5, cy = 23.5
    cfg = O.vol_cfg(voxel_size=0.02)
    pose = O.IDENTITY.copy()
    pose[9:] = (shift, shift, 0.0)
    d = np.full((k.height, k.width), 0.3, np.float32)
    rgb = np.full((k.height, k.width, 3), 90, np.uint8)
    rgb[:, ::2] = 200
    ov, gv = pair(cfg)
    for _ in range(3):
        ov.carve(d, k, pose)
        gv.carve(frame(k, d), pose)
        ov.allocate_for_frame(d, k, pose)
        gv.allocate_for_frame(frame(k, d), pose)
        ov.integrate(d, rgb, k, pose)
        gv.integrate(frame(k, d, rgb), pose)
    assert_volumes_identical(ov, gv)
    # the layer really sits on ties (the fast path's 1e-9 margin catches them)
    coords, _ = ov.export()
    s = cfg.voxel_size
    ties = 0
    for c in coords:
        v = (np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij"), -1).reshape(-1, 3)
             + 8 * c[:3])
        ctr = (v + 0.5) * s
        z = ctr[:, 2]
        on = (np.abs(z - 0.25) < 1e-12)
        x = k.fx * (ctr[on, 0] - shift) / z[on] + k.cx
        ties += int(np.sum(np.abs(x - np.floor(x) - 0.5) <= 1e-9))
    assert ties > 0


def test_allocation_640x480_keys_and_occupancy():
    """Full-size frame of the bench scene: bit-exact key set and hash occupancy."""
    s = O.Scene(scenes.bench_script(frames=3))
    r = s.render(1)
    pose = s.camera(1)[1]
    ov, gv = pair(O.vol_cfg())
    ov.allocate_for_frame(r["depth"], s.k, pose)
    gv.allocate_for_frame(frame(s.k, r["depth"]), pose)
    assert ov.num_blocks() == gv.num_blocks() > 1000
    oc, _ = canonical(*ov.export(False))
    gc, _ = canonical(*gv.export(False))
    assert (oc == gc).all()
    assert (ov.hash_occupancy(gv.hash_capacity()) == gv.hash_occupancy()).all()
    ov.integrate(r["depth"], r["rgb"], s.k, pose)
    gv.integrate(frame(s.k, r["depth"], r["rgb"]), pose)
    assert_volumes_identical(ov, gv, check_occupancy=False)


def test_block_budget_raises():
    gv = G.TsdfVolume(G.volume_config(voxel_size=0.02, max_blocks=4))
    for x in range(4):
        assert gv.allocate_block((x, 0, 0))
    with pytest.raises(G.ResourceLimitError):
        gv.allocate_block((4, 0, 0))
    assert not gv.allocate_block((0, 0, 0))
    k = O.small_intrinsics()
    gv2 = G.TsdfVolume(G.volume_config(voxel_size=0.02, max_blocks=3))
    with pytest.raises(G.ResourceLimitError):
        gv2.allocate_for_frame(frame(k, np.full((k.height, k.width), 0.5, np.float32)), O.IDENTITY)


def wavy_volumes(voxel=0.02, lo=(-0.4, -0.4, 0.0), hi=(0.4, 0.4, 0.8), weight=32):
    ov, gv = pair(O.vol_cfg(voxel_size=voxel, truncation=0.1))
    blocks, coords, rec = H.fill_voxels(voxel, 8, lo, hi, H.wavy_probe, H.wavy_probe_intensity, weight)
    for b in blocks:
        ov.allocate_block(b)
    gv.allocate_blocks(blocks)
    assert ov.set_voxels(coords, rec) == 0
    assert gv.set_voxels(coords, rec) == 0
    return ov, gv


def test_sampling_bitexact_all_modes():
    ov, gv = wavy_volumes()
    rng = np.random.default_rng(5)
    pts = np.concatenate([np.stack([rng.uniform(-0.45, 0.45, 3000), rng.uniform(-0.45, 0.45, 3000),
                                    rng.uniform(-0.05, 0.85, 3000)], 1),
                          # lattice-aligned points hit the brick-straddling gathers
                          (np.floor(rng.uniform(-20, 20, (500, 3))) + 0.5) * 0.02])
    for mode in range(5):
        ov_v, ov_g, ov_ok = ov.sample(pts, mode)
        gv_v, gv_g, gv_ok = gv.sample(pts, mode)
        assert (ov_ok == gv_ok).all(), mode
        assert ov_ok.sum() > 1000
        assert (ov_v[ov_ok] == gv_v[gv_ok]).all(), mode
        if mode >= 2:
            assert (ov_g[ov_ok] == gv_g[gv_ok]).all(), mode


def test_small_hash_long_probe_chains():
    """A hash table at load ~0.7 (2^12 slots): most lookups continue past their home
    slot (gather_corners' collision path, k_alloc's probe and CAS chains, the link
    records of displaced bricks). Fused voxels, hash occupancy and samples stay
    bit-identical to the oracle's."""
    k = O.small_intrinsics(64, 48, 50.0)
    ocfg = O.vol_cfg(voxel_size=0.005, max_blocks=3200)  # ~2850 bricks
    gc = gcfg(ocfg)
    gc.hash_capacity = 1 << 12
    ov, gv = O.Volume(ocfg), G.TsdfVolume(gc)
    rng = np.random.default_rng(9)
    for i in range(4):
        d, rgb = wavy_frame(k, 20 + i)
        pose = H.small_pose(rng.uniform(-0.03, 0.03, 3), rng.uniform(-1, 1, 3), rng.uniform(-0.05, 0.05))
        ov.carve(d, k, pose)
        gv.carve(frame(k, d), pose)
        ov.allocate_for_frame(d, k, pose)
        gv.allocate_for_frame(frame(k, d), pose)
        ov.integrate(d, rgb, k, pose)
        gv.integrate(frame(k, d, rgb), pose)
    assert gv.hash_capacity() == 1 << 12 and gv.num_blocks() > 0.5 * (1 << 12)
    assert_volumes_identical(ov, gv)
    assert all(v == 0 for v in gv.check().values())
    pts = np.stack([rng.uniform(-0.3, 0.3, 4000), rng.uniform(-0.25, 0.25, 4000), rng.uniform(0.2, 0.8, 4000)], 1)
    for mode in range(5):
        ov_v, ov_g, ov_ok = ov.sample(pts, mode)
        gv_v, gv_g, gv_ok = gv.sample(pts, mode)
        assert (ov_ok == gv_ok).all(), mode
        assert ov_ok.sum() > 200, mode
        assert (ov_v[ov_ok] == gv_v[gv_ok]).all(), mode
        if mode >= 2:
            assert (ov_g[ov_ok] == gv_g[gv_ok]).all(), mode
    # the tracking kernel's gathers through the same chains
    o = ov.linearize(d, rgb, k, pose, O.reg_cfg(color_weight=0.025))
    g = gv.linearize(frame(k, d, rgb), pose, G.registration_config(color_weight=0.025))
    assert o["valid"] == g["valid"] > 500
    np.testing.assert_allclose(g["H"], o["H"], rtol=1e-9, atol=1e-9 * np.abs(o["H"]).max())
    np.testing.assert_allclose(g["b"], o["b"], rtol=1e-9, atol=1e-9 * np.abs(o["b"]).max())


def test_voxel_handle_roundtrip_and_export():
    ov, gv = wavy_volumes()
    coords = np.array([[0, 0, 10], [-3, 5, 20], [100, 100, 100]], np.int32)
    a, fa = ov.get_voxels(coords)
    b, fb = gv.get_voxels(coords)
    assert (fa == fb).all() and a.tobytes() == b.tobytes()
    assert_volumes_identical(ov, gv)


# ------------------------------------------------------------------ registration
@pytest.fixture(scope="module")
def corner():
    s = O.Scene(scenes.corner_scene())
    r = s.render(0)
    view = s.camera(0)[1]
    ov, gv = pair(O.vol_cfg(voxel_size=0.02, truncation=0.1))
    ov.allocate_for_frame(r["depth"], s.k, view)
    ov.integrate(r["depth"], r["rgb"], s.k, view)
    gv.allocate_for_frame(frame(s.k, r["depth"]), view)
    gv.integrate(frame(s.k, r["depth"], r["rgb"]), view)
    assert_volumes_identical(ov, gv)
    init = H.compose(view, H.small_pose((0.03, -0.02, 0.04), (1.0, 1.0, 0.0), 3.0 * math.pi / 180))
    return dict(s=s, r=r, view=view, ov=ov, gv=gv, init=init)


def test_linearize_normal_equations(corner):
    c = corner
    for cw in (0.0, 0.025):
        o = c["ov"].linearize(c["r"]["depth"], c["r"]["rgb"], c["s"].k, c["init"], O.reg_cfg(color_weight=cw))
        g = c["gv"].linearize(frame(c["s"].k, c["r"]["depth"], c["r"]["rgb"]), c["init"],
                              G.registration_config(color_weight=cw))
        assert o["valid"] == g["valid"] > 1000
        np.testing.assert_allclose(g["H"], o["H"], rtol=1e-9, atol=1e-9 * np.abs(o["H"]).max())
        np.testing.assert_allclose(g["b"], o["b"], rtol=1e-9, atol=1e-9 * np.abs(o["b"]).max())
        assert g["error"] == pytest.approx(o["error"], rel=1e-9)


def test_evaluate_depth_error_residual_image_bitexact(corner):
    c = corner
    k = c["s"].k
    mask = np.zeros((k.height, k.width), np.uint8)
    mask[:, :20] = 1
    e_o, sq_o, v_o = c["ov"].evaluate_depth_error(c["r"]["depth"], k, c["init"], mask)
    e_g, sq_g, v_g = c["gv"].evaluate_depth_error(frame(k, c["r"]["depth"]), c["init"], mask)
    assert (v_o == v_g).all() and (sq_o == sq_g).all()
    assert e_g == pytest.approx(e_o, rel=1e-12)
    ce_o = c["ov"].evaluate_color_error(c["r"]["depth"], c["r"]["rgb"], k, c["init"])
    ce_g = c["gv"].evaluate_color_error(frame(k, c["r"]["depth"], c["r"]["rgb"]), c["init"])
    assert ce_g == pytest.approx(ce_o, rel=1e-12)


@pytest.mark.parametrize("cw", [0.0, 0.025])
def test_register_matches_oracle(corner, cw):
    c = corner
    k = c["s"].k
    o = c["ov"].register(c["r"]["depth"], c["r"]["rgb"], k, c["init"], None, O.reg_cfg(color_weight=cw))
    g = c["gv"].register(frame(k, c["r"]["depth"], c["r"]["rgb"]), c["init"], None,
                         G.registration_config(color_weight=cw))
    dt, dr = pose_error(o["pose"], g["pose"])
    assert dt <= POSE_TOL_T and dr <= POSE_TOL_R
    assert g["iterations"] == o["iterations"]
    assert g["valid_residuals"] == o["valid_residuals"]
    assert g["converged"] == o["converged"]
    et, er = pose_error(c["view"], g["pose"])  # test_registration.cpp:184-204
    assert et < 5e-3 and er < 0.5 * math.pi / 180


@pytest.mark.parametrize("levels", [1, 2, 4, 5])
def test_register_pyramid_depths(corner, levels):
    """Register with other pyramid depths than the default 3 (the per-level
    ranges, intrinsics and images the kernel stages per level). Five levels of
    the 64x48 image leave a 4x3 top level: too few residuals, TrackingLost on
    both sides."""
    c = corner
    k = c["s"].k
    if levels == 5:
        with pytest.raises(O.TrackingLost):
            c["ov"].register(c["r"]["depth"], c["r"]["rgb"], k, c["init"], None, O.reg_cfg(pyramid_levels=5))
        with pytest.raises(G.TrackingLostError):
            c["gv"].register(frame(k, c["r"]["depth"], c["r"]["rgb"]), c["init"], None,
                             G.registration_config(pyramid_levels=5))
        return
    o = c["ov"].register(c["r"]["depth"], c["r"]["rgb"], k, c["init"], None, O.reg_cfg(pyramid_levels=levels))
    g = c["gv"].register(frame(k, c["r"]["depth"], c["r"]["rgb"]), c["init"], None,
                         G.registration_config(pyramid_levels=levels))
    dt, dr = pose_error(o["pose"], g["pose"])
    assert dt <= POSE_TOL_T and dr <= POSE_TOL_R
    assert g["iterations"] == o["iterations"] and g["valid_residuals"] == o["valid_residuals"]


def test_register_with_mask_ignores_corruption(corner):  # test_registration.cpp:220-262
    c = corner
    k = c["s"].k
    clean = c["r"]["depth"]
    corrupted = clean.copy()
    mask = np.zeros((k.height, k.width), np.uint8)
    sl = (slice(None), slice(0, k.width // 3))
    corrupted[sl] = np.where(corrupted[sl] > 0, corrupted[sl] + np.float32(0.05), corrupted[sl])
    mask[sl] = 1
    a = c["gv"].register(frame(k, clean, c["r"]["rgb"]), c["init"], mask)
    b = c["gv"].register(frame(k, corrupted, c["r"]["rgb"]), c["init"], mask)
    assert (a["pose"] == b["pose"]).all()
    o = c["ov"].register(corrupted, c["r"]["rgb"], k, c["init"], mask)
    dt, dr = pose_error(o["pose"], b["pose"])
    assert dt <= POSE_TOL_T and dr <= POSE_TOL_R
    assert (o["res_sq"] == b["res_sq"]).all() or np.abs(o["res_sq"] - b["res_sq"]).max() < 1e-6


def test_tracking_lost():
    gv = G.TsdfVolume(G.volume_config(voxel_size=0.025))
    blocks, coords, rec = H.fill_voxels(0.025, 8, (-0.2, -0.2, 0.4), (0.2, 0.2, 0.6), H.wavy_probe)
    gv.allocate_blocks(blocks)
    gv.set_voxels(coords, rec)
    k = O.small_intrinsics()
    with pytest.raises(G.TrackingLostError):
        gv.register(frame(k, np.full((k.height, k.width), 3.0, np.float32)), O.IDENTITY)


# ------------------------------------------------------------------ mask
def test_mask_stages_bitexact_random():
    rng = np.random.default_rng(3)
    h, w = 96, 128
    depth = (1.0 + 0.5 * (rng.random((h, w)) < 0.3) + 0.003 * rng.standard_normal((h, w))).astype(np.float32)
    depth[rng.random((h, w)) < 0.05] = 0
    sq = (rng.random((h, w)) * 0.01).astype(np.float32)
    valid = (rng.random((h, w)) < 0.9).astype(np.uint8)
    for cfg in (O.mask_cfg(), O.mask_cfg(erode_radius=1, dilate_radius=3, connectivity=8, theta=0.02)):
        gc = G.mask_config(gamma=cfg.gamma, truncation=cfg.truncation, theta=cfg.theta,
                           erode_radius=cfg.erode_radius, dilate_radius=cfg.dilate_radius,
                           connectivity=cfg.connectivity)
        assert (O.build_mask(sq, valid, depth, cfg) == G.build_mask(sq, valid, depth, gc)).all()
    seeds = (rng.random((h, w)) < 0.01).astype(np.uint8)
    for theta in (0.007, 0.05, 0.6):
        for conn in (4, 8):
            assert (O.floodfill(seeds, depth, theta, conn) == G.floodfill_depth(seeds, depth, theta, conn)).all()
    m = (rng.random((h, w)) < 0.6).astype(np.uint8)
    for r in (0, 1, 2, 3):
        assert (O.erode(m, r) == G.erode(m, r)).all()
        assert (O.dilate(m, r) == G.dilate(m, r)).all()
    assert (O.threshold(sq, valid) == G.threshold_residuals(sq, valid)).all()


def test_mask_kats():  # test_mask.cpp fixtures on the CUDA path
    sq = np.array([[0.005, 0.0051, 1.0, 0.0049]], np.float32)
    valid = np.array([[1, 1, 0, 1]], np.uint8)
    assert G.threshold_residuals(sq, valid).tolist() == [[0, 1, 0, 0]]
    d = np.zeros((5, 5), np.float32)
    d[:, :3] = 1.0
    d[:, 3:] = 1.5
    s = np.zeros((5, 5), np.uint8)
    s[1, 1] = 1
    exp = np.zeros((5, 5), np.uint8)
    exp[:, :3] = 1
    assert (G.floodfill_depth(s, d, 0.007) == exp).all()
    d = np.array([[2.0, 2.012, 2.03]], np.float32)
    assert G.floodfill_depth(np.array([[1, 0, 0]], np.uint8), d, 0.007).tolist() == [[1, 1, 0]]
    d = np.ones((2, 2), np.float32)
    d[0, 1] = d[1, 0] = 2.0
    s = np.array([[1, 0], [0, 0]], np.uint8)
    assert G.floodfill_depth(s, d, 0.007, 4)[1, 1] == 0 and G.floodfill_depth(s, d, 0.007, 8)[1, 1] == 1
    # a long serpentine region forces many global floodfill rounds
    h, w = 64, 256
    d = np.full((h, w), 2.0, np.float32)
    for y in range(0, h, 4):
        d[y, :] = 1.0
        d[y:y + 4, (w - 1) if (y // 4) % 2 == 0 else 0] = 1.0
    s = np.zeros((h, w), np.uint8)
    s[0, 0] = 1
    assert (O.floodfill(s, d, 0.007) == G.floodfill_depth(s, d, 0.007)).all()


# ------------------------------------------------------------------ raycast
def test_raycast_bitexact():
    k = O.small_intrinsics(48, 36, 40.0)
    ov, gv = pair(O.vol_cfg(voxel_size=0.02))
    for i in range(3):
        d, rgb = wavy_frame(k, 10 + i)
        ov.allocate_for_frame(d, k, O.IDENTITY)
        ov.integrate(d, rgb, k, O.IDENTITY)
        gv.allocate_for_frame(frame(k, d), O.IDENTITY)
        gv.integrate(frame(k, d, rgb), O.IDENTITY)
    view = H.small_pose((0.01, -0.02, 0.0), (0, 1, 0), 0.05)
    a = ov.raycast(view, k)
    b = gv.raycast(view, gk(k))
    assert (a > 0).sum() > 100
    assert (a == b).all()


def test_save_load_roundtrip(tmp_path):
    _, gv = wavy_volumes()
    p = str(tmp_path / "vol.bin")
    gv.save(p)
    lv = G.TsdfVolume.load(p)
    a = canonical(*gv.export())
    b = canonical(*lv.export())
    assert (a[0] == b[0]).all() and a[1].tobytes() == b[1].tobytes()
    with open(p, "rb") as f:
        assert f.read(8) == b"TSDFVOL\0"


# ------------------------------------------------------------------ pipeline
def run_both(script, n=None, dynamics=True, reg_threads=8):
    s = O.Scene(script)
    n = n or len(s)
    frames = [s.render(i) for i in range(n)]
    op = O.Pipeline(O.pipe_cfg(refine=False, dynamics=dynamics, reg=O.reg_cfg(threads=reg_threads)))
    gp = G.Pipeline(G.pipeline_config(refine=False, dynamics=dynamics))
    out = []
    for f in frames:
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = gp.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"]))
        out.append((so, po, sg, pg))
    return s, frames, op, gp, out


def test_pipeline_static_scene_matches_oracle():
    s, frames, op, gp, out = run_both(scenes.pipeline_static_scene())
    for so, po, sg, pg in out:
        dt, dr = pose_error(po, pg)
        assert dt <= POSE_TOL_T and dr <= POSE_TOL_R
        for key in ("tracking_lost", "registrations", "iterations", "masked_pixels", "valid_residuals"):
            assert so[key] == sg[key], key
    assert gp.tracking_losses() == 0


@pytest.mark.parametrize("mover", [False, True])
def test_pipeline_acceptance_room(mover):
    """acceptance.cpp criteria 3/4 on the CUDA path plus per-frame pose parity."""
    s, frames, op, gp, out = run_both(scenes.room_script(with_mover=mover))
    worst = max(max(pose_error(po, pg)) for _, po, _, pg in out)
    assert worst <= 1e-4
    gt = [s.camera(i)[1] for i in range(len(s))]
    bound = 0.01 * (2 if mover else 1)
    assert H.ate_rmse([pg for *_, pg in out], gt) < bound
    assert gp.tracking_losses() == 0
    # the same criterion through the product's AteRmse (timestamp association, evaluation.cpp:26-62)
    rmse, _, pairs = G.ate_rmse(gp.trajectory(), [s.camera(i) for i in range(len(s))])
    assert pairs == len(s) == 30 and rmse < bound
    assert abs(rmse - H.ate_rmse([pg for *_, pg in out], gt)) < 1e-9


def test_pipeline_lockstep_volume_bitexact():
    """Lockstep mode: the CUDA mapping path fed the oracle's poses and masks
    produces a bit-identical volume (SURVEY §8d parity mode i)."""
    s = O.Scene(scenes.room_script(with_mover=True, frames=8))
    op = O.Pipeline(O.pipe_cfg(refine=False, reg=O.reg_cfg(threads=8)))
    gv = G.TsdfVolume(gcfg(O.vol_cfg()))
    for i in range(len(s)):
        f = s.render(i)
        st, pose = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        fr = frame(s.k, f["depth"], f["rgb"])
        if i == 0:
            gv.allocate_for_frame(fr, pose)
            gv.integrate(fr, pose)
            continue
        mask = op.last_mask(s.k)
        gv.carve(fr, pose)
        gv.allocate_for_frame(fr, pose, mask)
        gv.integrate(fr, pose, mask)
    assert_volumes_identical(op.volume(), gv)


def test_pipeline_bench_scene_640x480_prefix():
    """The bench workload (C2, 640x480, 1 cm, moving boxes): first frames
    against the oracle, poses and stats."""
    s, frames, op, gp, out = run_both(scenes.bench_script(), n=4)
    for so, po, sg, pg in out:
        dt, dr = pose_error(po, pg)
        assert dt <= POSE_TOL_T and dr <= POSE_TOL_R
        assert so["registrations"] == sg["registrations"]
        assert abs(so["masked_pixels"] - sg["masked_pixels"]) <= 0.001 * 640 * 480


def test_process_frames_batch_matches_single():
    """rf_pipeline_process_frames (frames enqueued back to back) gives the same
    poses, stats and volume as frame-by-frame ProcessFrame, over more frames
    than one batch holds."""
    s = O.Scene(scenes.room_script(with_mover=True, width=160, height=120, frames=70))
    frames = [s.render(i) for i in range(len(s))]
    cfg = G.pipeline_config(refine=False, volume=G.volume_config(voxel_size=0.02, max_blocks=200000))
    a, b = G.Pipeline(cfg), G.Pipeline(cfg)
    single = [a.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"])) for f in frames]
    stats, poses = b.process_frames([frame(s.k, f["depth"], f["rgb"], f["timestamp"]) for f in frames])
    for (sa, pa), sb, pb in zip(single, stats, poses):
        assert np.array_equal(pa, pb)
        for key in ("frame_index", "tracking_lost", "registrations", "iterations", "masked_pixels", "valid_residuals",
                    "final_error"):
            assert sa[key] == sb[key], key
    assert np.array_equal(a.trajectory()[1], b.trajectory()[1])
    ca, va = canonical(*a.volume().export())
    cb, vb = canonical(*b.volume().export())
    assert (ca == cb).all() and va.tobytes() == vb.tobytes()


def test_pipeline_tracking_loss_single_and_batch():
    """A frame with no usable depth loses tracking (registration.cpp:228-231):
    the pose is held, nothing is integrated, later frames recover
    (pipeline.cpp:117-122) -- frame by frame against the oracle, and the batched
    call (loss handled on the device) identical to the single calls."""
    s = O.Scene(scenes.room_script(with_mover=False, width=160, height=120, frames=8))
    frames = [s.render(i) for i in range(len(s))]
    frames[4] = dict(frames[4], depth=np.zeros_like(frames[4]["depth"]))
    vc = O.vol_cfg(voxel_size=0.02, max_blocks=200000)
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=vc, reg=O.reg_cfg(threads=8)))
    cfg = G.pipeline_config(refine=False, volume=gcfg(vc))
    ga, gb = G.Pipeline(cfg), G.Pipeline(cfg)
    gframes = [frame(s.k, f["depth"], f["rgb"], f["timestamp"]) for f in frames]
    bstats, bposes = gb.process_frames(gframes)
    for i, f in enumerate(frames):
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = ga.process_frame(gframes[i])
        assert so["tracking_lost"] == sg["tracking_lost"] == bstats[i]["tracking_lost"], i
        assert max(pose_error(po, pg)) <= 1e-4
        assert np.array_equal(pg, bposes[i])
    assert bstats[4]["tracking_lost"] == 1 and np.array_equal(bposes[4], bposes[3])
    assert ga.tracking_losses() == gb.tracking_losses() == 1


def test_pipeline_nonfinite_and_negative_depth():
    """Depth pixels that are NaN, +inf, -inf, negative or zero are invalid
    (image.hpp:68 DepthValid: d > 0 and finite) everywhere on the path --
    allocation, integration, pyramid and registration -- so a frame sequence
    salted with them tracks and fuses as the oracle does, and the batched call
    matches the single calls."""
    s = O.Scene(scenes.room_script(with_mover=False, width=160, height=120, frames=6))
    frames = [s.render(i) for i in range(len(s))]
    rng = np.random.default_rng(7)
    bad = np.array([np.nan, np.inf, -np.inf, -1.0, 0.0], np.float32)
    for i in range(1, len(frames)):
        d = frames[i]["depth"].copy()
        idx = rng.choice(d.size, size=d.size // 20, replace=False)
        d.reshape(-1)[idx] = bad[rng.integers(0, len(bad), size=idx.size)]
        frames[i] = dict(frames[i], depth=d)
    vc = O.vol_cfg(voxel_size=0.02, max_blocks=200000)
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=vc, reg=O.reg_cfg(threads=8)))
    cfg = G.pipeline_config(refine=False, volume=gcfg(vc))
    ga, gb = G.Pipeline(cfg), G.Pipeline(cfg)
    gframes = [frame(s.k, f["depth"], f["rgb"], f["timestamp"]) for f in frames]
    bstats, bposes = gb.process_frames(gframes)
    for i, f in enumerate(frames):
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = ga.process_frame(gframes[i])
        assert so["tracking_lost"] == sg["tracking_lost"] == bstats[i]["tracking_lost"] == 0, i
        assert max(pose_error(po, pg)) <= 1e-4, i
        assert np.array_equal(pg, bposes[i]), i


@pytest.mark.parametrize("h,w", [(1, 1), (33, 45), (67, 101), (130, 37)])
def test_mask_stages_bitexact_ragged(h, w):
    """The mask stages on image sizes that are not multiples of the 32x32
    floodfill tile or of 4 bytes (the byte-wise row path), down to 1x1."""
    rng = np.random.default_rng(h * 1000 + w)
    depth = (1.0 + 0.5 * (rng.random((h, w)) < 0.3) + 0.003 * rng.standard_normal((h, w))).astype(np.float32)
    depth[rng.random((h, w)) < 0.05] = 0
    sq = (rng.random((h, w)) * 0.01).astype(np.float32)
    valid = (rng.random((h, w)) < 0.9).astype(np.uint8)
    for cfg in (O.mask_cfg(), O.mask_cfg(erode_radius=1, dilate_radius=3, connectivity=8, theta=0.02)):
        gc = G.mask_config(gamma=cfg.gamma, truncation=cfg.truncation, theta=cfg.theta,
                           erode_radius=cfg.erode_radius, dilate_radius=cfg.dilate_radius,
                           connectivity=cfg.connectivity)
        assert (O.build_mask(sq, valid, depth, cfg) == G.build_mask(sq, valid, depth, gc)).all()
    seeds = (rng.random((h, w)) < 0.02).astype(np.uint8)
    for theta in (0.007, 0.6):
        for conn in (4, 8):
            assert (O.floodfill(seeds, depth, theta, conn) == G.floodfill_depth(seeds, depth, theta, conn)).all()
    m = (rng.random((h, w)) < 0.6).astype(np.uint8)
    for r in (1, 3):
        assert (O.erode(m, r) == G.erode(m, r)).all()
        assert (O.dilate(m, r) == G.dilate(m, r)).all()


def test_mask_floodfill_atomic_worklist_path():
    """A frame whose floodfill tile flags do not fit in the tracking kernel's
    dynamic shared memory (8192 x 4608: 36864 tiles) takes the atomic
    worklist path of the floodfill (ff_flag_mode false); it must give the
    oracle's mask bit for bit like the flag path does at camera sizes."""
    rng = np.random.default_rng(21)
    h, w = 4608, 8192
    yy, xx = np.mgrid[0:h, 0:w]
    depth = np.zeros((h, w), np.float32)
    # depth-continuous bands the growth can run along, with gaps it cannot cross
    band = ((yy // 64) % 3) != 2
    depth[band] = (1.0 + 0.0005 * (xx[band] % 512) / 512.0).astype(np.float32)
    sq = np.zeros((h, w), np.float32)
    valid = band.astype(np.uint8)
    for _ in range(60):  # eroded-surviving seed blocks scattered over the bands
        cy, cx = int(rng.integers(0, h - 8)), int(rng.integers(0, w - 8))
        sq[cy:cy + 8, cx:cx + 8] = 0.05
    cfg = O.mask_cfg()
    gc = G.mask_config()
    om = O.build_mask(sq, valid, depth, cfg)
    gm = G.build_mask(sq, valid, depth, gc)
    assert om.sum() > 100000
    assert (om == gm).all()


def test_mask_wide_morphology_path():
    """Erosion / dilation radii beyond the tiled path's halo (kMorphMaxR = 8)
    run as separable passes through global memory; bit-exact as well."""
    rng = np.random.default_rng(8)
    h, w = 120, 200
    depth = (1.0 + 0.5 * (rng.random((h, w)) < 0.2) + 0.002 * rng.standard_normal((h, w))).astype(np.float32)
    sq = (rng.random((h, w)) * 0.004).astype(np.float32)
    sq[20:90, 30:150] = 0.02  # a large region that survives a wide erosion
    valid = (rng.random((h, w)) < 0.95).astype(np.uint8)
    valid[20:90, 30:150] = 1
    for er, dr, conn in ((9, 2, 4), (2, 11, 8), (10, 12, 8)):
        oc = O.mask_cfg(erode_radius=er, dilate_radius=dr, connectivity=conn)
        gc = G.mask_config(erode_radius=er, dilate_radius=dr, connectivity=conn)
        om, gm = O.build_mask(sq, valid, depth, oc), G.build_mask(sq, valid, depth, gc)
        assert om.sum() > 0 and (om == gm).all(), (er, dr, conn)
