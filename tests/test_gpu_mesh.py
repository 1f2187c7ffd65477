"""Marching cubes on the CUDA path (rf_volume_extract_mesh) against the
oracle's ExtractMesh (proj/src/mesh.cpp:50-181): identical vertex bytes,
colours and face indices, in the reference's order. test_mesh.cpp:43-148
properties (on-surface, outward, watertight) are checked on the GPU mesh too.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests import helpers as H
from tests.test_gpu_parity import gcfg, frame, pair

pytestmark = pytest.mark.gpu


def assert_meshes_identical(a, b):
    (va, ca, fa), (vb, cb, fb) = a, b
    assert va.shape == vb.shape, f"vertices {len(va)} vs {len(vb)}"
    assert fa.shape == fb.shape, f"faces {len(fa)} vs {len(fb)}"
    assert va.tobytes() == vb.tobytes(), "vertex positions differ"
    assert (ca == cb).all(), "vertex colours differ"
    assert (fa == fb).all(), "faces differ"


def test_sphere_mesh_matches_oracle_and_properties():  # test_mesh.cpp:43-126
    center, radius = np.array([0.1, -0.05, 0.4]), 0.25
    ov, gv = pair(O.vol_cfg(voxel_size=0.02, truncation=0.1))
    m = radius + 0.1
    blocks, coords, rec = H.fill_voxels(0.02, 8, center - m, center + m,
                                        lambda p: float(np.linalg.norm(p - center) - radius),
                                        lambda p: 60.0 + 100.0 * (p[2] - 0.15) / 0.5)
    for b in blocks:
        ov.allocate_block(b)
    gv.allocate_blocks(blocks)
    assert ov.set_voxels(coords, rec) == 0 and gv.set_voxels(coords, rec) == 0
    for mw in (1, 2):
        assert_meshes_identical(ov.extract_mesh(mw), gv.extract_mesh(mw))
    v, c, f = gv.extract_mesh(1)
    assert len(v) > 1000 and len(f) > 1000
    r = np.linalg.norm(v.astype(np.float64) - center, axis=1)
    assert np.abs(r - radius).max() < 0.25 * 0.02
    a, b, cc = (v[f[:, i]].astype(np.float64) for i in range(3))
    n = np.cross(b - a, cc - a)
    assert (np.sum(n * ((a + b + cc) / 3 - center), 1) > 0).mean() > 0.99
    edges = {}
    for tri in f:
        for i in range(3):
            e = tuple(sorted((int(tri[i]), int(tri[(i + 1) % 3]))))
            edges[e] = edges.get(e, 0) + 1
    assert all(cnt == 2 for cnt in edges.values())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_volume_mesh_order_bitexact(seed):
    """Random signs, weights and colours over a ragged brick set: every cube
    configuration, incomplete cells, missing neighbour bricks, zero and equal
    sdf pairs (the 1e-12 denominator branch) and cross-brick edge ownership."""
    rng = np.random.default_rng(seed)
    ov, gv = pair(O.vol_cfg(voxel_size=0.01, truncation=0.05))
    cand = np.array([(x, y, z) for z in range(-2, 2) for y in range(-2, 2) for x in range(-2, 2)], np.int32)
    blocks = cand[rng.random(len(cand)) < 0.7]
    for b in blocks:
        ov.allocate_block(tuple(int(t) for t in b))
    gv.allocate_blocks(blocks)
    coords = (blocks[:, None, :] * 8 + np.stack(np.meshgrid(np.arange(8), np.arange(8), np.arange(8),
                                                          indexing="ij"), -1).reshape(-1, 3)[None]).reshape(-1, 3)
    coords = coords.astype(np.int32)
    rec = np.zeros(len(coords), dtype=H.VOXEL_DTYPE)
    sdf = rng.normal(0.0, 0.02, len(coords)).astype(np.float32)
    sdf[rng.random(len(coords)) < 0.05] = 0.0
    sdf[rng.random(len(coords)) < 0.05] = np.float32(0.01)
    rec["sdf"] = sdf
    rec["weight"] = rng.integers(0, 5, len(coords))
    rec["weight"][rng.random(len(coords)) < 0.6] = 10
    for ch in "rgb":
        rec[ch] = rng.integers(0, 256, len(coords))
    assert ov.set_voxels(coords, rec) == 0 and gv.set_voxels(coords, rec) == 0
    for mw in (0, 2, 5):
        om = ov.extract_mesh(mw)
        assert len(om[2]) > (100 if mw < 5 else 10)
        assert_meshes_identical(om, gv.extract_mesh(mw))


def test_integrated_room_mesh_bitexact():
    """Mesh of a volume fused from rendered frames (lockstep poses): the C4
    export path at a small size."""
    s = O.Scene(scenes.room_script(with_mover=False, frames=4))
    ov, gv = pair(O.vol_cfg(voxel_size=0.02))
    for i in range(len(s)):
        f = s.render(i)
        pose = s.camera(i)[1]
        ov.allocate_for_frame(f["depth"], s.k, pose)
        ov.integrate(f["depth"], f["rgb"], s.k, pose)
        gv.allocate_for_frame(frame(s.k, f["depth"]), pose)
        gv.integrate(frame(s.k, f["depth"], f["rgb"]), pose)
    om = ov.extract_mesh(2)
    assert len(om[2]) > 10000
    assert_meshes_identical(om, gv.extract_mesh(2))


def test_empty_volume_and_ply(tmp_path):
    gv = G.TsdfVolume(G.volume_config(voxel_size=0.02))
    v, c, f = gv.extract_mesh()
    assert v.shape == (0, 3) and f.shape == (0, 3)
    center, radius = np.array([0.0, 0.0, 0.5]), 0.1
    H.fill_volume(gv, center - 0.15, center + 0.15, lambda p: float(np.linalg.norm(p - center) - radius))
    p = tmp_path / "m.ply"
    v, c, f = gv.extract_mesh(2, ply_path=p)
    data = p.read_bytes()
    head, body = data.split(b"end_header\n", 1)
    assert f"element vertex {len(v)}".encode() in head and f"element face {len(f)}".encode() in head
    assert len(body) == 15 * len(v) + 13 * len(f)
    vb = np.frombuffer(body[:15 * len(v)], dtype=np.dtype([("p", "<f4", 3), ("c", "u1", 3)]))
    assert (vb["p"] == v).all() and (vb["c"] == c).all()
    fb = np.frombuffer(body[15 * len(v):], dtype=np.dtype([("n", "u1"), ("i", "<i4", 3)]))
    assert (fb["n"] == 3).all() and (fb["i"] == f).all()
