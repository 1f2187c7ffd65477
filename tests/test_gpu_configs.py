"""BASELINE.json workloads as parity cases on the CUDA path, each against the
oracle on the same oracle-rendered frames (the pattern of
proj/tests/acceptance.cpp:287-408):

  C1 -- static room, 640x480, 1 cm: the whole 50-frame sequence free-running;
  C2 -- room + 2 moving boxes, the whole 200-frame bench sequence free-running;
  C3 -- the large scene (6 x 2 x 6 m room + props) at 0.5 cm with the 4M-entry
        (2^22) hash: 30 frames lockstep (volume, pool order and occupancy
        bit-exact) and free-running (poses, counts);
  C4 -- 1280x720 with K = (1050, 1050, 639.5, 359.5), 3 levels: 30 frames
        lockstep + free-running, then ExtractMesh bit-exact.

Free-running bars: poses <= 1e-4 m / 1e-4 rad per frame (north_star), and the
per-frame registrations, LM iterations, masked pixels and tracking losses
equal to the oracle's.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests.test_gpu_mesh import assert_meshes_identical
from tests.test_gpu_parity import assert_volumes_identical, frame, gcfg, pose_error

pytestmark = pytest.mark.gpu

COUNTS = ("registrations", "iterations", "masked_pixels", "tracking_lost")


def config_volume(name):
    c = scenes.BENCH_CONFIGS[name]
    return O.vol_cfg(voxel_size=c["voxel"], max_blocks=c.get("max_blocks", 1000000)), c.get("hash_capacity")


def run(name, n, lockstep=False):
    """Oracle pipeline and the CUDA pipeline on the same frames; with
    `lockstep`, a CUDA volume also carves / allocates / integrates with the
    oracle's poses and masks (pipeline.cpp:25-29)."""
    s = O.Scene(scenes.config_script(name))
    ocfg, cap = config_volume(name)
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=ocfg, reg=O.reg_cfg(threads=16), threads=16))
    gc = gcfg(ocfg)
    if cap:
        gc.hash_capacity = cap
    gp = G.Pipeline(G.pipeline_config(refine=False, volume=gc))
    gv = G.TsdfVolume(gc) if lockstep else None
    worst, mism = 0.0, {k: 0 for k in COUNTS}
    for i in range(n):
        f = s.render(i)
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = gp.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"]))
        worst = max(worst, *pose_error(po, pg))
        for k in COUNTS:
            mism[k] += int(so[k] != sg[k])
        if gv is not None:
            fr = frame(s.k, f["depth"], f["rgb"])
            if i == 0:
                gv.allocate_for_frame(fr, po)
                gv.integrate(fr, po)
            else:
                mask = op.last_mask(s.k)
                gv.carve(fr, po)
                gv.allocate_for_frame(fr, po, mask)
                gv.integrate(fr, po, mask)
    return op, gp, gv, worst, mism


@pytest.mark.parametrize("name,n", [("C1", 50), ("C2", 200)])
def test_whole_sequence_free_running(name, n):
    op, gp, _, worst, mism = run(name, n)
    assert worst <= 1e-4, worst
    assert mism == {k: 0 for k in COUNTS}, mism
    assert gp.tracking_losses() == op.losses() == 0
    assert all(v == 0 for v in gp.volume().check().values())
    assert len(gp.trajectory()[0]) == n


def test_c3_large_scene_half_centimetre_4m_hash():
    op, gp, gv, worst, mism = run("C3", 30, lockstep=True)
    assert gv.hash_capacity() == 1 << 22
    ov = op.volume()
    assert ov.num_blocks() > 100000
    assert_volumes_identical(ov, gv)  # key set, voxels and the occupied-slot bitmap at 2^22
    oc, _ = ov.export(False)
    gc, _ = gv.export(False)
    assert (oc == gc).all()  # pool (allocation) order too
    assert all(v == 0 for v in gv.check().values()) and all(v == 0 for v in gp.volume().check().values())
    assert worst <= 1e-4, worst
    assert mism == {k: 0 for k in COUNTS}, mism


def test_c4_1280x720_mesh_export():
    s = O.Scene(scenes.config_script("C4"))
    assert (s.k.width, s.k.height, s.k.fx, s.k.cx, s.k.cy) == (1280, 720, 1050.0, 639.5, 359.5)
    op, gp, gv, worst, mism = run("C4", 30, lockstep=True)
    assert_volumes_identical(op.volume(), gv)
    assert worst <= 1e-4, worst
    assert mism == {k: 0 for k in COUNTS}, mism
    om = op.volume().extract_mesh(2)
    assert len(om[2]) > 50000
    assert_meshes_identical(om, gv.extract_mesh(2))


def test_1920x1080_pixel_cache_overflow():
    """At 1920x1080 a thread meets 37 pixel steps at level 0, more than the
    pixel cache holds (32 steps in its 96 KB): the steps beyond it reload their
    inputs every pass. Poses and counts still match the oracle frame by frame."""
    s = O.Scene(scenes.room_script(with_mover=True, width=1920, height=1080, frames=5))
    op = O.Pipeline(O.pipe_cfg(refine=False, reg=O.reg_cfg(threads=16), threads=16))
    gp = G.Pipeline(G.pipeline_config(refine=False))
    worst, mism = 0.0, {k: 0 for k in COUNTS}
    for i in range(len(s)):
        f = s.render(i)
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = gp.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"]))
        worst = max(worst, *pose_error(po, pg))
        for k in COUNTS:
            mism[k] += int(so[k] != sg[k])
    assert worst <= 1e-4, worst
    assert mism == {k: 0 for k in COUNTS}, mism
    assert all(v == 0 for v in gp.volume().check().values())
