"""The opt-in extensions north_star names and the reference lacks (SURVEY.md
preamble, deltas 1-2): Huber-weighted residuals in registration
(SPEC.md:276 says the reference has no robust kernel; registration.cpp:72-95
is plain least squares) and a free-space term in the dynamics mask
(dynamics_mask.cpp:98-104 has none). Both default to off, and off reproduces
the reference; these CPU tests pin the oracle's restatement of each
extension, which the -m gpu tests (test_gpu_extensions.py) then hold the CUDA
path to.
"""
import numpy as np

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes


def test_defaults_are_off():
    assert O.reg_cfg().huber_depth == O.reg_cfg().huber_color == 0.0
    assert O.mask_cfg().free_space == 0.0
    assert G.registration_config().huber_depth == G.registration_config().huber_color == 0.0
    assert G.mask_config().free_space == 0.0
    c = G.pipeline_config()
    assert c.registration.huber_depth == 0.0 and c.mask.free_space == 0.0


def max_drift(huber_depth, frames=15):
    """Dynamics mask off, so the moving box's pixels stay in the objective:
    the worst per-frame translation error against the ground-truth camera."""
    s = O.Scene(scenes.room_script(with_mover=True, width=160, height=120, frames=frames))
    p = O.Pipeline(O.pipe_cfg(refine=False, dynamics=False, reg=O.reg_cfg(threads=8, huber_depth=huber_depth),
                              threads=8))
    g0 = np.linalg.inv(O.pose_matrix(s.camera(0)[1]))
    worst = 0.0
    for i in range(len(s)):
        f = s.render(i)
        _, pose = p.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        rel = g0 @ O.pose_matrix(s.camera(i)[1])
        worst = max(worst, float(np.linalg.norm(O.pose_matrix(np.asarray(pose))[:3, 3] - rel[:3, 3])))
    return worst


def test_huber_damps_a_moving_object():
    plain, robust = max_drift(0.0), max_drift(0.02)
    assert plain > 0.025  # the box drags the least-squares track (3.4 cm here)
    assert robust < 0.6 * plain  # Huber at 2 cm halves it (2.0 cm)


def test_huber_threshold_above_every_residual_is_plain_least_squares():
    k = O.small_intrinsics(64, 48, 50.0)
    vol = O.Volume(O.vol_cfg(voxel_size=0.02))
    d = np.full((k.height, k.width), 1.0, np.float32)
    d[:, 20:40] = 0.9
    rgb = np.full((k.height, k.width, 3), 90, np.uint8)
    rgb[10:30] = 200
    vol.allocate_for_frame(d, k, O.IDENTITY)
    vol.integrate(d, rgb, k, O.IDENTITY)
    pose = O.pose_array(t=(0.004, -0.003, 0.01))
    a = vol.linearize(d, rgb, k, pose, O.reg_cfg())
    b = vol.linearize(d, rgb, k, pose, O.reg_cfg(huber_depth=1e3, huber_color=1e3))
    for key in ("H", "b"):
        assert (np.asarray(a[key]) == np.asarray(b[key])).all()
    assert a["error"] == b["error"] and a["valid"] == b["valid"] > 500
    # below the residuals: every row is down-weighted and the cost grows linearly
    c = vol.linearize(d, rgb, k, pose, O.reg_cfg(huber_depth=1e-4))
    assert c["valid"] == a["valid"]
    assert np.abs(np.asarray(c["H"])).max() < np.abs(np.asarray(a["H"])).max()


def test_free_space_seeds_are_a_superset():
    rng = np.random.default_rng(5)
    h, w = 60, 80
    depth = (1.0 + 0.001 * rng.standard_normal((h, w))).astype(np.float32)
    depth[20:40, 30:55] = 0.8  # an object in front: residuals in model free space
    sq = (rng.random((h, w)) * 0.0008).astype(np.float32)
    valid = rng.choice(np.array([1, 3], np.uint8), size=(h, w))
    valid[rng.random((h, w)) < 0.05] = 0
    sq[20:40, 30:55] = 0.002  # below gamma * truncation^2 = 0.005, above 0.03^2
    valid[20:40, 30:55] = 3
    sq[5:15, 5:15] = 0.02  # a residual blob the reference threshold catches on its own
    valid[5:15, 5:15] = 1
    off = O.build_mask(sq, valid, depth, O.mask_cfg())
    on = O.build_mask(sq, valid, depth, O.mask_cfg(free_space=0.03))
    assert off[10, 10] and not off[30, 40]
    assert (on >= off).all() and on[30, 40] and on[20:40, 30:55].all()
    # the seeds: the reference threshold, or bit 1 (positive residual) above free_space^2
    t = O.build_mask(sq, valid, depth, O.mask_cfg(free_space=0.03, erode_radius=0, dilate_radius=0, theta=1e-9))
    sq64 = sq.astype(np.float64)
    expect = ((valid != 0) & (sq64 > 0.5 * 0.1 * 0.1)) | (((valid & 2) != 0) & (sq64 > 0.03 * 0.03))
    assert (t == expect).all()
