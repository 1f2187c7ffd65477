"""Boundary entry points added for parity with the reference interface:
LinearizeResult::degenerate (registration.cpp:128-140), BuildPyramid
(registration.hpp:42), FindBlock as one hash probe (tsdf_volume.cpp:59-62),
and the C++ host layer's reference-style voxel handles."""
import math
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from tests import helpers as H
from tests.test_cpp_host import CXX, LIBDIR, ROOT
from tests.test_gpu_parity import frame, gcfg, wavy_volumes

pytestmark = pytest.mark.gpu


def plane_pair():
    vc = O.vol_cfg(voxel_size=0.02, truncation=0.1)
    ov, gv = O.Volume(vc), G.TsdfVolume(gcfg(vc))
    blocks, coords, rec = H.fill_voxels(0.02, 8, (-1.0, -1.0, 0.3), (1.0, 1.0, 0.7), lambda p: p[2] - 0.5)
    for b in blocks:
        ov.allocate_block(b)
    gv.allocate_blocks(blocks)
    assert ov.set_voxels(coords, rec) == 0 and gv.set_voxels(coords, rec) == 0
    return ov, gv


def test_plane_is_degenerate():  # test_registration.cpp:142-151
    ov, gv = plane_pair()
    k = O.small_intrinsics()
    d = np.full((k.height, k.width), 0.5, np.float32)
    g = gv.linearize(frame(k, d), O.IDENTITY, G.registration_config(color_weight=0.0))
    o = ov.linearize(d, None, k, O.IDENTITY, O.reg_cfg(color_weight=0.0))
    assert g["valid"] == o["valid"] > 0
    assert g["degenerate"] and o["degenerate"]


def test_textured_surface_is_not_degenerate():
    ov, gv = wavy_volumes()
    k = O.small_intrinsics(64, 48, 50.0)
    d, rgb = H.make_frame(k, lambda u, v: 0.45 + 0.04 * math.sin(0.4 * u) * math.cos(0.3 * v),
                          lambda u, v: 110.0 + 60.0 * math.sin(0.25 * u + 0.1 * v))
    g = gv.linearize(frame(k, d, rgb), O.IDENTITY)
    o = ov.linearize(d, rgb, k, O.IDENTITY)
    assert g["valid"] == o["valid"] > 100
    assert g["degenerate"] == o["degenerate"]
    # nothing valid: degenerate by definition
    z = np.zeros((k.height, k.width), np.float32)
    assert gv.linearize(frame(k, z), O.IDENTITY)["degenerate"]


def test_pyramid_kat():  # test_registration.cpp:50-77
    k = O.small_intrinsics(8, 4, 10.0)
    d, rgb = H.make_frame(k, lambda u, v: 1.0 + u + 8.0 * v, lambda u, v: 10.0 * u + v)
    d[1, 2] = 0.0
    mask = np.zeros((4, 8), np.uint8)
    mask[2, 5] = 1
    pyr = G.build_pyramid(frame(k, d, rgb), mask, 3)
    assert pyr[1]["depth"].shape == (2, 4) and pyr[2]["depth"].shape == (1, 2)
    assert pyr[1]["intrinsics"].fx == pytest.approx(5.0)
    assert pyr[1]["depth"][0, 0] == pytest.approx(1.0)
    assert pyr[1]["depth"][0, 1] == pytest.approx(3.0)
    assert pyr[1]["intensity"][0, 0] == pytest.approx((0 + 10 + 1 + 11) / 4.0, rel=1e-6)
    assert pyr[1]["mask"][1, 2] == 1 and pyr[1]["mask"][0, 0] == 0 and pyr[2]["mask"][0, 1] == 1
    with pytest.raises(ValueError):
        G.build_pyramid(frame(k, d, rgb), None, 0)


@pytest.mark.parametrize("w,h,levels", [(640, 480, 3), (101, 67, 4), (33, 17, 2), (5, 3, 1)])
def test_pyramid_bitexact_vs_oracle(w, h, levels):
    rng = np.random.default_rng(w * h)
    k = O.small_intrinsics(w, h, 0.8 * w)
    d = rng.uniform(0.2, 4.0, (h, w)).astype(np.float32)
    d[rng.random((h, w)) < 0.15] = 0.0
    d[rng.random((h, w)) < 0.01] = np.nan
    rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    mask = (rng.random((h, w)) < 0.05).astype(np.uint8)
    o = O.build_pyramid(d, rgb, k, levels, mask)
    g = G.build_pyramid(frame(k, d, rgb), mask, levels)
    for l in range(levels):
        assert g[l]["depth"].tobytes() == o[l]["depth"].tobytes(), l
        assert g[l]["intensity"].tobytes() == o[l]["intensity"].tobytes(), l
        assert (g[l]["mask"] == o[l]["mask"]).all(), l
        ki = g[l]["intrinsics"]
        assert (ki.fx, ki.fy, ki.cx, ki.cy) == tuple(o[l]["intr"])
    # no colour, no mask
    g2 = G.build_pyramid(frame(k, d), None, levels)
    assert g2[-1]["intensity"] is None and g2[-1]["mask"] is None
    assert g2[-1]["depth"].tobytes() == o[-1]["depth"].tobytes()


def test_find_block_single_probe():
    ov, gv = wavy_volumes()
    oc, ovox = ov.export()
    for i in [0, len(oc) // 2, len(oc) - 1]:
        got = gv.find_block(oc[i])
        assert got is not None and got.tobytes() == ovox[i].tobytes()
    assert gv.find_block((999, 999, 999)) is None
    vox = ovox[0].copy()
    vox["weight"] = 77
    assert gv.write_block(oc[0], vox)
    assert gv.find_block(oc[0])["weight"].tolist() == [77] * 512
    assert not gv.write_block((999, 999, 999), vox)


def test_cpp_host_voxel_handles(tmp_path):
    exe = str(tmp_path / "host_volume_demo")
    subprocess.run([CXX, "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_volume_demo.cpp"), "-L", LIBDIR, "-lrefusion_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True, capture_output=True, text=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and r.stdout.count("ok") >= 14


def test_device_frames_checked_and_ordered():
    """CUDA-tensor frames go to the library as raw pointers: wrong dtype,
    layout or device is refused, and work torch queued for them is complete
    before the library's own stream reads them (refusion_b200.h stream contract)."""
    import torch

    s_k = O.small_intrinsics(64, 48, 50.0)
    k = G.intrinsics(s_k.fx, s_k.fy, s_k.cx, s_k.cy, s_k.width, s_k.height, s_k.depth_scale)
    d = torch.full((48, 64), 0.5, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        G.Frame(d.double(), None, k).c()
    with pytest.raises(ValueError):
        G.Frame(torch.full((64, 48), 0.5, device="cuda").t(), None, k).c()  # non-contiguous
    with pytest.raises(ValueError):
        G.Frame(d, torch.zeros((48, 64, 3), dtype=torch.float32, device="cuda"), k).c()
    # produced on torch's stream right before the call: the volume sees the final values
    ov, gv = plane_pair()
    big = torch.empty((48, 64), dtype=torch.float32, device="cuda")
    for _ in range(50):
        big.fill_(0.1)
    big.fill_(0.5)
    g = gv.linearize(G.Frame(big, None, k), O.IDENTITY, G.registration_config(color_weight=0.0))
    o = ov.linearize(np.full((48, 64), 0.5, np.float32), None, s_k, O.IDENTITY, O.reg_cfg(color_weight=0.0))
    assert g["valid"] == o["valid"] and g["depth_error"] == pytest.approx(o["depth_error"], rel=1e-12, abs=1e-18)
