"""Refinement-window pipeline (refine on, window 10) over a few C2 frames, for
an ncu launch list of IntegrateFront's kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_02082_b200 import api, scenes, synth  # noqa: E402


def main(n=40):
    scene = synth.parse(scenes.config_script("C2"))
    k = scene.intrinsics
    d = torch.empty((n, k.height, k.width), dtype=torch.float32, device="cuda")
    c = torch.empty((n, k.height, k.width, 3), dtype=torch.uint8, device="cuda")
    lab = torch.empty((n, k.height, k.width), dtype=torch.uint8, device="cuda")
    for i in range(n):
        synth.render(scene, i, d[i], c[i], lab[i])
    torch.cuda.synchronize()
    p = api.Pipeline(api.pipeline_config(refine=True, window=10))
    for i in range(n):
        p.process_frame(api.Frame(depth=d[i], rgb=c[i], intrinsics=k, timestamp=i / 30.0))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
