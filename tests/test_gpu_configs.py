"""BASELINE.json configs beyond the bench line, as parity cases on the CUDA
path (a few frames each; the oracle runs the same frames):

  C3 -- 0.5 cm voxels with the 4M-entry (2^22) hash: occupancy bitmap and
        volume bit-exact in lockstep, pipeline poses <= 1e-4.
  C4 -- 1280x720 with K = (1050, 1050, 639.5, 359.5), 3 pyramid levels, mesh
        export: lockstep volume + ExtractMesh bit-exact, pipeline poses.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests.test_gpu_mesh import assert_meshes_identical
from tests.test_gpu_parity import assert_volumes_identical, frame, gcfg, pose_error

pytestmark = pytest.mark.gpu


def lockstep(script, ocfg, n, cap=None):
    """Oracle pipeline drives the poses and masks; the CUDA volume carves,
    allocates and integrates the same frames (pipeline.cpp:25-29)."""
    s = O.Scene(script)
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=ocfg, reg=O.reg_cfg(threads=8), threads=8))
    gc = gcfg(ocfg)
    if cap:
        gc.hash_capacity = cap
    gv = G.TsdfVolume(gc)
    gp = G.Pipeline(G.pipeline_config(refine=False, volume=gcfg(ocfg)))
    worst = 0.0
    for i in range(n):
        f = s.render(i)
        st, pose = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        _, pg = gp.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"]))
        worst = max(worst, *pose_error(pose, pg))
        fr = frame(s.k, f["depth"], f["rgb"])
        if i == 0:
            gv.allocate_for_frame(fr, pose)
            gv.integrate(fr, pose)
            continue
        mask = op.last_mask(s.k)
        gv.carve(fr, pose)
        gv.allocate_for_frame(fr, pose, mask)
        gv.integrate(fr, pose, mask)
    return op, gv, worst


def test_c3_half_centimetre_4m_hash():
    ocfg = O.vol_cfg(voxel_size=0.005, max_blocks=4000000)
    op, gv, worst = lockstep(scenes.bench_script(dynamic=True, frames=200, seed=43), ocfg, 3, cap=1 << 22)
    assert gv.hash_capacity() == 1 << 22
    assert op.volume().num_blocks() > 20000
    assert_volumes_identical(op.volume(), gv)  # includes the occupied-slot bitmap at 2^22
    assert worst <= 1e-4


def test_c4_1280x720_mesh_export():
    ocfg = O.vol_cfg()
    script = scenes.bench_script(dynamic=True, width=1280, height=720, frames=1000, seed=44)
    s = O.Scene(script)
    assert (s.k.width, s.k.height, s.k.fx, s.k.cx, s.k.cy) == (1280, 720, 1050.0, 639.5, 359.5)
    op, gv, worst = lockstep(script, ocfg, 3)
    assert_volumes_identical(op.volume(), gv)
    assert worst <= 1e-4
    om = op.volume().extract_mesh(2)
    assert len(om[2]) > 50000
    assert_meshes_identical(om, gv.extract_mesh(2))
