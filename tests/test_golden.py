"""Golden fixture tests/golden/acceptance_room_160x120.npz (made by
tests/golden/make_golden.py from the KAT-pinned oracle): the oracle must keep
reproducing it (CPU), and the CUDA path must match it from the fixture's own
input bytes, without the oracle (GPU)."""
import hashlib
import os

import numpy as np
import pytest

from paper_1905_02082_b200 import api as G

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "acceptance_room_160x120.npz")


def load():
    return dict(np.load(GOLDEN))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def canonical(coords, vox):
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    return coords[order], vox[order]


def intrinsics(g):
    fx, fy, cx, cy, w, h, ds = g["intrinsics"]
    return G.intrinsics(fx, fy, cx, cy, int(w), int(h), ds)


def masks(g):
    n = len(g["pose"])
    h, w = int(g["intrinsics"][5]), int(g["intrinsics"][4])
    return [np.unpackbits(g["mask_bits"][i])[: h * w].reshape(h, w) for i in range(n)]


def test_oracle_reproduces_golden():
    from tests.golden import make_golden

    g = load()
    fresh = make_golden.generate()
    for key in ("depth", "rgb", "timestamp", "gt_pose", "intrinsics", "pose", "counts", "mask_bits"):
        np.testing.assert_array_equal(fresh[key], g[key], err_msg=key)
    for key in ("volume_bricks", "volume_sha", "mesh_counts", "mesh_sha", "raycast_sha"):
        assert np.array_equal(np.asarray(fresh[key]), g[key]), key


@pytest.mark.gpu
def test_cuda_pipeline_matches_golden():
    g = load()
    k = intrinsics(g)
    cfg = G.pipeline_config(refine=False, volume=G.volume_config(voxel_size=0.02, max_blocks=200000))
    p = G.Pipeline(cfg)
    ms = masks(g)
    for i in range(len(g["pose"])):
        st, pose = p.process_frame(G.Frame(g["depth"][i], g["rgb"][i], k, float(g["timestamp"][i])))
        d = pose - g["pose"][i]
        assert np.abs(d[9:]).max() <= 1e-4 and np.abs(d[:9]).max() <= 1e-4, i
        assert [st["registrations"], st["iterations"], st["masked_pixels"], st["tracking_lost"]] == \
            g["counts"][i].tolist(), i
        if i > 0:
            got = p.last_mask_image(k)
            assert got is not None and np.array_equal(got.astype(bool), ms[i].astype(bool)), i


@pytest.mark.gpu
def test_cuda_lockstep_volume_mesh_raycast_match_golden():
    """Carve / AllocateForFrame / Integrate on the golden poses and masks:
    bit-identical volume, ExtractMesh and raycast (SHA-256 of the bytes)."""
    g = load()
    k = intrinsics(g)
    v = G.TsdfVolume(G.volume_config(voxel_size=0.02, max_blocks=200000))
    ms = masks(g)
    for i in range(len(g["pose"])):
        f = G.Frame(g["depth"][i], g["rgb"][i], k)
        m = ms[i] if i > 0 else None
        if i > 0:
            v.carve(f, g["pose"][i])
        v.allocate_for_frame(f, g["pose"][i], m)
        v.integrate(f, g["pose"][i], m)
    c, vox = canonical(*v.export())
    assert len(c) == int(g["volume_bricks"]) and sha(c, vox) == str(g["volume_sha"])
    mv, mc, mf = v.extract_mesh(2)
    assert [len(mv), len(mf)] == g["mesh_counts"].tolist() and sha(mv, mc, mf) == str(g["mesh_sha"])
    assert sha(v.raycast(g["pose"][-1], k)) == str(g["raycast_sha"])
