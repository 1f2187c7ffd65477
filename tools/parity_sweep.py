"""Whole-sequence parity of the CUDA pipeline against the oracle on the
BASELINE.json workloads (oracle-rendered frames, both sides consume identical
bytes; refine off like the acceptance config): per-frame pose difference,
identical iteration / registration / masked-pixel counts, ATE of each side
against the ground-truth trajectory (product AteRmse), and the final volumes
(brick key sets, voxel agreement)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1905_02082_b200 import api as G, scenes  # noqa: E402
from tests import helpers as H  # noqa: E402


def gk(k):
    return G.intrinsics(k.fx, k.fy, k.cx, k.cy, k.width, k.height, k.depth_scale)


def sweep(name, script, threads=16):
    t0 = time.time()
    s = O.Scene(script)
    op = O.Pipeline(O.pipe_cfg(refine=False, threads=threads, reg=O.reg_cfg(threads=threads)))
    gp = G.Pipeline(G.pipeline_config(refine=False))
    worst_t = worst_r = 0.0
    mism = {"iterations": 0, "registrations": 0, "masked_pixels": 0, "tracking_lost": 0}
    for i in range(len(s)):
        f = s.render(i)
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = gp.process_frame(G.Frame(f["depth"], f["rgb"], gk(s.k), f["timestamp"]))
        d = H.compose(H.inverse(po), pg)
        worst_t = max(worst_t, float(np.linalg.norm(d[9:])))
        worst_r = max(worst_r, float(np.linalg.norm(po[:9] - pg[:9])))  # ||R_o - R_g||_F (acos is noisy at 0)
        for k in mism:
            mism[k] += int(so[k] != sg[k])
    gt = [s.camera(i) for i in range(len(s))]
    ate_g = G.ate_rmse(gp.trajectory(), gt)[0]
    ate_o = G.ate_rmse((np.array([t for t, _ in op.trajectory]), np.array([p for _, p in op.trajectory])), gt)[0]
    oc, ov = op.volume().export()
    gc, gv = gp.volume().export()
    ko = {tuple(c) for c in oc}
    kg = {tuple(c) for c in gc}
    oi = {tuple(c): i for i, c in enumerate(oc)}
    common = [(oi[tuple(c)], j) for j, c in enumerate(gc) if tuple(c) in oi]
    a = ov[[i for i, _ in common]]
    b = gv[[j for _, j in common]]
    same = float(np.mean(a.view(np.uint64) == b.view(np.uint64)))
    both = (a["weight"] > 0) & (b["weight"] > 0)
    dsdf = float(np.max(np.abs(a["sdf"][both] - b["sdf"][both]))) if both.any() else 0.0
    print(f"{name}: {len(s)} frames, worst pose diff {worst_t:.2e} m / ||dR||_F {worst_r:.2e}, "
          f"count mismatches {mism}, ATE gpu {ate_g * 1e3:.3f} mm / oracle {ate_o * 1e3:.3f} mm, "
          f"bricks {len(gc)} vs {len(oc)} (sym diff {len(ko ^ kg)}), voxels bit-identical {same * 100:.3f}%, "
          f"max |sdf diff| where both observed {dsdf:.2e}, {time.time() - t0:.0f} s", flush=True)


def main():
    sweep("C1", scenes.config_script("C1"))
    sweep("C2", scenes.config_script("C2"))
    sweep("acceptance RoomScript(true) 320x240", scenes.room_script(with_mover=True))


if __name__ == "__main__":
    main()
