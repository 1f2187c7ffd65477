"""Frames/s of the pipeline with the reference's default depth-refinement window
(refine on, window 10) on the C2 workload, for DESIGN.md (not a bench line)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_02082_b200 import api, scenes, synth  # noqa: E402


def main(n=120):
    scene = synth.parse(scenes.bench_script(dynamic=True, frames=200, seed=43))
    k = scene.intrinsics
    d = torch.empty((n, k.height, k.width), dtype=torch.float32, device="cuda")
    c = torch.empty((n, k.height, k.width, 3), dtype=torch.uint8, device="cuda")
    lab = torch.empty((n, k.height, k.width), dtype=torch.uint8, device="cuda")
    for i in range(n):
        synth.render(scene, i, d[i], c[i], lab[i])
    torch.cuda.synchronize()
    for refine in (False, True):
        p = api.Pipeline(api.pipeline_config(refine=refine, window=10))
        frames = [api.Frame(depth=d[i], rgb=c[i], intrinsics=k, timestamp=i / 30.0) for i in range(n)]
        for f in frames[:20]:
            p.process_frame(f)
        t0 = time.perf_counter()
        for f in frames[20:]:
            p.process_frame(f)
        dt = time.perf_counter() - t0
        print(f"refine={refine}: {(n - 20) / dt:.1f} frames/s (per-frame calls)")


if __name__ == "__main__":
    main()
