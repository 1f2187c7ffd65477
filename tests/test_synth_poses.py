"""The GPU renderer's host side (paper_1905_02082_b200/synth.py) computes the
camera and per-primitive world-to-object poses in the reference's operation
order (synth.cpp:26-45, 155-158; geometry.hpp:78-96): they must equal the
oracle's RenderFrame poses bit for bit (CPU test; the per-pixel kernel is
compared in tests/test_gpu_synth.py)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import scenes, synth


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_renderer_poses_bit_identical(name):
    text = scenes.config_script(name)
    o, g = O.Scene(text), synth.parse(text)
    assert len(o) == len(g)
    for i in range(len(o)):
        t, pose = o.camera(i)
        gt, gpose = g.camera[i]
        assert gt == t
        assert np.asarray(gpose).tobytes() == pose.tobytes(), f"camera {i}"
        for j, prim in enumerate(g.prims):
            R, tr = synth._inverse(*synth._pose_at(prim, gt))
            assert np.concatenate([R.reshape(9), tr]).tobytes() == o.world_to_object(j, t).tobytes(), (i, j)
