"""Generates tests/golden/acceptance_room_160x120.npz. It is a self-contained
fixture of the reference's acceptance room (acceptance.cpp:82-113,
RoomScript(true): static room plus the moving sphere), 160x120, first 5 frames.

Inputs: the oracle-rendered depth and colour bytes, plus the ground-truth
camera poses.

Outputs of the oracle pipeline (refine off, the acceptance config):

- per frame: pose, registrations, iterations, masked-pixel count, tracking
  loss, and the dynamics mask (packed bits);
- for the final volume, driven in lockstep (oracle poses and masks): the brick
  count and a SHA-256 of the canonical (x, y, z)-sorted bricks and voxels;
- ExtractMesh(min_weight 2) of that volume: counts and SHA-256;
- the raycast depth of the last pose: SHA-256.

The oracle itself is pinned by the reference's KATs (tests/test_oracle_*.py).
This fixture freezes its outputs, so the CUDA path can be checked on the GPU box
without the oracle. It also guards the oracle against drift
(tests/test_golden.py).

Usage: python tests/golden/make_golden.py  (needs the oracle built: make -C oracle)
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1905_02082_b200 import scenes  # noqa: E402

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "acceptance_room_160x120.npz")
FRAMES = 5
VOXEL = 0.02


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def canonical(coords, vox):
    order = np.lexsort((coords[:, 2], coords[:, 1], coords[:, 0]))
    return coords[order], vox[order]


def script():
    return scenes.room_script(with_mover=True, width=160, height=120, frames=FRAMES)


def volume_cfg():
    return O.vol_cfg(voxel_size=VOXEL, max_blocks=200000)


def generate():
    s = O.Scene(script())
    k = s.k
    frames = [s.render(i) for i in range(FRAMES)]
    op = O.Pipeline(O.pipe_cfg(refine=False, volume=volume_cfg(), reg=O.reg_cfg(threads=8), threads=8))
    lock = O.Volume(volume_cfg())
    out = dict(depth=np.stack([f["depth"] for f in frames]).astype(np.float32),
               rgb=np.stack([f["rgb"] for f in frames]).astype(np.uint8),
               timestamp=np.array([f["timestamp"] for f in frames]),
               gt_pose=np.stack([s.camera(i)[1] for i in range(FRAMES)]),
               intrinsics=np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_scale]))
    poses, counts, masks = [], [], []
    for i, f in enumerate(frames):
        st, pose = op.process_frame(f["depth"], f["rgb"], k, f["timestamp"])
        poses.append(pose)
        counts.append([st["registrations"], st["iterations"], st["masked_pixels"], st["tracking_lost"]])
        mask = op.last_mask(k) if i > 0 else None
        masks.append(np.packbits(mask.astype(bool)) if mask is not None else np.packbits(np.zeros(k.width * k.height, bool)))
        if i > 0:
            lock.carve(f["depth"], k, pose)
        lock.allocate_for_frame(f["depth"], k, pose, mask)
        lock.integrate(f["depth"], f["rgb"], k, pose, mask)
    c, v = canonical(*lock.export())
    mv, mc, mf = lock.extract_mesh(2)
    ray = lock.raycast(poses[-1], k)
    out.update(pose=np.stack(poses), counts=np.array(counts, np.int64), mask_bits=np.stack(masks),
               volume_bricks=np.int64(len(c)), volume_sha=sha(c, v),
               mesh_counts=np.array([len(mv), len(mf)], np.int64), mesh_sha=sha(mv, mc, mf),
               raycast_sha=sha(ray))
    return out


if __name__ == "__main__":
    g = generate()
    np.savez_compressed(PATH, **g)
    print(f"wrote {PATH} ({os.path.getsize(PATH)} bytes): {g['volume_bricks']} bricks, "
          f"{g['mesh_counts'][0]} vertices, masked {g['counts'][:, 2].tolist()}")
