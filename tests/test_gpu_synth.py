"""rf_synth_render (the GPU workload renderer, csrc/rf_synth.cu) against
RenderFrame (synth.cpp:136-203, oracle restatement) with the depth noise off:
depth, colour and dynamic labels must be identical bytes. (With noise on, the
GPU draws counter-based normals where the reference draws mt19937 +
std::normal_distribution; bench.py therefore feeds both arms the oracle's
bytes, and this test pins everything else the renderer computes.)"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1905_02082_b200 import scenes, synth

pytestmark = pytest.mark.gpu


def noise_free(text):
    return "\n".join("noise 0 0.0" if ln.startswith("noise") else ln for ln in text.splitlines()) + "\n"


@pytest.mark.parametrize("name,frames", [("C1", [0, 17, 49]), ("C2", [0, 1, 66, 133, 199])])
def test_synth_render_matches_renderframe_noise_free(name, frames):
    text = noise_free(scenes.config_script(name))
    o, g = O.Scene(text), synth.parse(text)
    k = g.intrinsics
    H, W = k.height, k.width
    d = torch.empty((H, W), dtype=torch.float32, device="cuda")
    c = torch.empty((H, W, 3), dtype=torch.uint8, device="cuda")
    lab = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    dynamic_px = 0
    for i in frames:
        ref = o.render(i)
        dynamic_px += int(ref["labels"].sum())
        synth.render(g, i, d, c, lab)
        torch.cuda.synchronize()
        gd, gc, gl = d.cpu().numpy(), c.cpu().numpy(), lab.cpu().numpy()
        assert ref["depth"].tobytes() == ref["true_depth"].tobytes()  # noise off: depth == true depth
        assert (gd.view(np.uint32) == ref["depth"].view(np.uint32)).all(), \
            f"frame {i}: {(gd != ref['depth']).sum()} depth pixels differ"
        assert (gc == ref["rgb"]).all(), f"frame {i}: {(gc != ref['rgb']).any(-1).sum()} colour pixels differ"
        assert (gl == ref["labels"]).all(), f"frame {i}: labels differ"
    assert (dynamic_px > 0) == (name == "C2")  # the moving boxes are in view of the sampled C2 frames
