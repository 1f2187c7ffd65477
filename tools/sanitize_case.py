"""A small end-to-end workload for compute-sanitizer (tools/sanitize.sh):
every kernel family on small sizes -- the persistent tracking kernel (grid
barrier, flagged-line all-reduce, LM, mask, floodfill), ordered allocation
(atomicCAS claims + atomicMin ordinals + ranked assignment), cull + link
records (concurrent link writers), fused carve/integrate, raycast, marching
cubes, BuildPyramid, an overflow with its recovery, and the batched path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1905_02082_b200 import api as G  # noqa: E402
from paper_1905_02082_b200 import scenes  # noqa: E402


def main():
    s = O.Scene(scenes.room_script(with_mover=True, width=96, height=72, frames=6))
    k = s.k
    gk = G.intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_scale)
    frames = [s.render(i) for i in range(len(s))]
    gf = [G.Frame(f["depth"], f["rgb"], gk, f["timestamp"]) for f in frames]
    cfg = G.pipeline_config(refine=False, volume=G.volume_config(voxel_size=0.02, max_blocks=20000))
    p = G.Pipeline(cfg)
    for f in gf[:3]:
        p.process_frame(f)
    p.process_frames(gf[3:])  # batched submission
    vol = p.volume()
    n = vol.num_blocks()
    v, c, fa = vol.extract_mesh(2)
    pose = p.trajectory()[1][-1]
    d = vol.raycast(pose, gk)
    pyr = G.build_pyramid(gf[0], (frames[0]["labels"] > 0).astype(np.uint8), 3)
    # refinement window on (window fusion kernels)
    pr = G.Pipeline(G.pipeline_config(refine=True, window=3, volume=G.volume_config(voxel_size=0.02,
                                                                                     max_blocks=20000)))
    for f in gf:
        pr.process_frame(f)
    pr.finalize()
    # an overflowing allocation and its recovery
    small = G.Pipeline(G.pipeline_config(refine=False, volume=G.volume_config(voxel_size=0.02, max_blocks=50)))
    try:
        small.process_frames(gf)
    except G.ResourceLimitError:
        pass
    print(f"sanitize case ok: {n} bricks, mesh {len(v)} vertices, raycast {int((d > 0).sum())} hits, "
          f"pyramid {pyr[2]['depth'].shape}, overflow pipeline {small.volume().num_blocks()} bricks")


if __name__ == "__main__":
    main()
