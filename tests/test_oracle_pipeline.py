"""Pins the oracle pipeline to proj/tests/test_pipeline.cpp and the end-to-end
acceptance criteria 3-5 (proj/tests/acceptance.cpp:287-480)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import scenes
from tests import helpers as H


@pytest.fixture(scope="module")
def static_scene():
    s = O.Scene(scenes.pipeline_static_scene())
    frames = [s.render(i) for i in range(len(s))]
    gt = [s.camera(i)[1] for i in range(len(s))]
    return s, frames, gt


def fast_cfg(**kw):  # test_pipeline.cpp:58-63 (refinement window 3)
    return O.pipe_cfg(refine=kw.pop("refine", True), window=3, **kw)


def run(cfg, s, frames):
    p = O.Pipeline(cfg)
    for f in frames:
        p.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
    p.finalize()
    return p


def test_static_scene_tracks(static_scene):  # test_pipeline.cpp:84-117
    s, frames, gt = static_scene
    p = run(fast_cfg(), s, frames)
    assert p.losses() == 0
    assert H.ate_rmse([t[1] for t in p.trajectory], gt) < 0.01
    px = s.k.width * s.k.height
    conv = 0
    for st in p.stats:
        assert not st["tracking_lost"]
        conv += st["converged"]
        assert st["masked_pixels"] < px / 100
        if st["frame_index"] > 0:
            assert st["registrations"] >= 1 and st["valid_residuals"] > px / 2
    assert conv + 2 >= len(p.stats)
    assert p.volume().num_blocks() > 100


def test_reruns_and_threads_identical(static_scene):  # test_pipeline.cpp:119-156
    s, frames, _ = static_scene
    a = run(fast_cfg(), s, frames)
    b = run(fast_cfg(), s, frames)
    c = run(fast_cfg(threads=2), s, frames)
    for x in (b, c):
        for (_, pa), (_, pb) in zip(a.trajectory, x.trajectory):
            assert (pa == pb).all()
        ea, eb = a.volume().export(), x.volume().export()
        assert (ea[0] == eb[0]).all() and ea[1].tobytes() == eb[1].tobytes()
    for sa, sb in zip(a.stats, b.stats):
        assert sa["iterations"] == sb["iterations"] and sa["final_error"] == sb["final_error"]


def test_dynamics_disabled_single_registration(static_scene):  # test_pipeline.cpp:158-171
    s, frames, _ = static_scene
    p = run(fast_cfg(dynamics=False), s, frames)
    for st in p.stats:
        assert st["masked_pixels"] == 0
        if st["frame_index"] > 0:
            assert st["registrations"] == 1
    assert p.losses() == 0


def test_tracking_loss_holds_pose(static_scene):  # test_pipeline.cpp:214-240
    s, frames, _ = static_scene
    p = O.Pipeline(fast_cfg(refine=False))
    p.process_frame(frames[0]["depth"], frames[0]["rgb"], s.k)
    p.process_frame(frames[1]["depth"], frames[1]["rgb"], s.k)
    nb = p.volume().num_blocks()
    held = p.trajectory[-1][1]
    st, pose = p.process_frame(np.zeros_like(frames[2]["depth"]), frames[2]["rgb"], s.k)
    assert st["tracking_lost"] and not st["converged"] and st["registrations"] == 0
    assert p.losses() == 1 and p.volume().num_blocks() == nb and (pose == held).all()
    st, _ = p.process_frame(frames[2]["depth"], frames[2]["rgb"], s.k)
    assert not st["tracking_lost"] and p.losses() == 1


def test_first_frame_identity(static_scene):  # test_pipeline.cpp:242-253
    s, frames, _ = static_scene
    p = O.Pipeline(fast_cfg())
    st, pose = p.process_frame(frames[0]["depth"], frames[0]["rgb"], s.k)
    assert st["registrations"] == 0 and st["converged"] and (pose == O.IDENTITY).all()
    assert p.volume().num_blocks() > 0


def test_intrinsics_mismatch_rejected(static_scene):  # test_pipeline.cpp:255-265
    s, frames, _ = static_scene
    p = O.Pipeline(fast_cfg())
    bad = O.OIntr(0.0, 40, 31.5, 23.5, 64, 48, 5000)
    with pytest.raises(ValueError):
        p.process_frame(frames[0]["depth"], frames[0]["rgb"], bad)


@pytest.mark.slow
def test_acceptance_static_and_dynamic_room():  # acceptance.cpp:287-408 (criteria 3 and 4)
    ates = {}
    for mover in (False, True):
        s = O.Scene(scenes.room_script(with_mover=mover))
        frames = [s.render(i) for i in range(len(s))]
        gt = [s.camera(i)[1] for i in range(len(s))]
        cfg = O.pipe_cfg(refine=False, reg=O.reg_cfg(threads=8))
        p = O.Pipeline(cfg)
        masks = []
        for f in frames:
            p.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
            masks.append(p.last_mask(s.k))
        p.finalize()
        assert p.losses() == 0
        ates[mover] = H.ate_rmse([t[1] for t in p.trajectory], gt)
        if mover:
            rec, fp = [], []
            for f, m in zip(frames, masks):
                g = f["labels"] != 0
                mm = (m != 0) if m is not None else np.zeros_like(g)
                if g.sum():
                    rec.append((mm & g).sum() / g.sum())
                fp.append((mm & ~g).sum() / max(1, (~g).sum()))
            assert np.mean(rec) >= 0.9
            assert np.mean(fp) <= 0.1
    assert ates[False] < 0.01
    assert ates[True] <= 2 * ates[False]


def test_acceptance_carve_reversion():  # acceptance.cpp:412-480 (criterion 5)
    vol = O.Volume(O.vol_cfg())
    k = O.small_intrinsics(64, 48, 60.0)
    center, radius = np.array([0.0, 0.0, 1.0]), 0.25

    def obj_depth(u, v):
        d = np.array([(u - k.cx) / k.fx, (v - k.cy) / k.fy, 1.0])
        a, b, c = d @ d, -2.0 * d @ center, center @ center - radius * radius
        disc = b * b - 4 * a * c
        if disc > 0:
            z = (-b - math.sqrt(disc)) / (2 * a)
            if z > 0.2:
                return z
        return 2.5

    d_obj, rgb = H.make_frame(k, obj_depth, lambda u, v: 128.0)
    d_wall, _ = H.make_frame(k, lambda u, v: 2.5, lambda u, v: 128.0)
    for _ in range(10):
        vol.allocate_for_frame(d_obj, k, O.IDENTITY)
        vol.integrate(d_obj, rgb, k, O.IDENTITY)
    coords, vox = vol.export()
    side = 8
    offs = np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij"), -1).reshape(-1, 3)[:, ::-1]
    vc = (coords[:, None, :] * side + offs[None]).reshape(-1, 3)
    vv = vox.reshape(-1)
    centers = (vc + 0.5) * 0.01
    sel = (vv["weight"] >= 1) & (np.abs(vv["sdf"]) < 0.05) & (np.linalg.norm(centers - center, axis=1) < radius + 0.1)
    obj = vc[sel]
    assert len(obj) > 0
    needed = None
    for n in range(1, 31):
        vol.carve(d_wall, k, O.IDENTITY)
        v, _ = vol.get_voxels(obj)
        if needed is None and (v["sdf"] > 0.05).all():
            needed = n
    assert needed is not None
