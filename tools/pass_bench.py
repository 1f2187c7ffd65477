"""Per-pass cost of the tracking kernel's Jacobian passes on the C2 workload
(rf_diag_pass_bench): builds the model from the first frames of the bench
sequence, then times `iters` passes per pyramid level at a fixed pose inside
one launch. Use RF_LIB_PATH to compare library variants."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_02082_b200 import _lib as L  # noqa: E402
from paper_1905_02082_b200 import api, scenes, synth  # noqa: E402


def main(frames=30, iters=200):
    lib = L.load()
    cfgd = scenes.BENCH_CONFIGS["C2"]
    scene = synth.parse(scenes.bench_script(dynamic=cfgd["dynamic"], frames=cfgd["frames"], seed=cfgd["seed"]))
    k = scene.intrinsics
    H, W = k.height, k.width
    depth = torch.empty((frames + 1, H, W), dtype=torch.float32, device="cuda")
    rgb = torch.empty((frames + 1, H, W, 3), dtype=torch.uint8, device="cuda")
    lab = torch.empty((frames + 1, H, W), dtype=torch.uint8, device="cuda")
    for i in range(frames + 1):
        synth.render(scene, i, depth[i], rgb[i], lab[i])
    p = api.Pipeline(api.pipeline_config(refine=False))
    pose = None
    for i in range(frames):
        _, pose = p.process_frame(api.Frame(depth=depth[i], rgb=rgb[i], intrinsics=k, timestamp=i / 30.0))
    vol = p.volume()
    f = api.Frame(depth=depth[frames], rgb=rgb[frames], intrinsics=k).c()
    out = {}
    for level in (0, 1, 2):
        us = C.c_double()
        acc = (C.c_double * 30)()
        L.check(lib.rf_diag_pass_bench(vol.h, C.byref(f), (C.c_double * 12)(*pose), level, iters, C.c_double(0.025),
                                       C.byref(us), acc))
        out[level] = (us.value, acc[29])
    print(" ".join(f"L{l}: {v[0]:.2f} us ({int(v[1])} px)" for l, v in out.items()), flush=True)


if __name__ == "__main__":
    main()
