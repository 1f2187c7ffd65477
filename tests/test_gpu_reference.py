"""The CUDA pipeline against the REFERENCE itself (oracle/_ref: the
unmodified /root/reference sources built with oracle/ref_shim), not only
against the restatement: the C2 bench sequence frame by frame (poses within
1e-4 m / rad, identical registrations, LM iterations, masked pixels), then the
final block set. Skipped where oracle/_ref was not built."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import reference as R
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests.test_gpu_parity import frame, pose_error

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]


def test_cuda_pipeline_vs_reference_c2():
    s = R.Scene(scenes.config_script("C2"))
    k = s.k
    rp = R.Pipeline(O.pipe_cfg(refine=False, threads=16, reg=O.reg_cfg(threads=16)))
    gp = G.Pipeline(G.pipeline_config(refine=False))
    worst = 0.0
    for i in range(40):
        f = s.render(i)
        sr, pr = rp.process_frame(f["depth"], f["rgb"], k, i / 30.0)
        sg, pg = gp.process_frame(frame(k, f["depth"], f["rgb"], i / 30.0))
        worst = max(worst, *pose_error(pr, pg))
        for key in ("tracking_lost", "registrations", "iterations", "masked_pixels"):
            assert sr[key] == sg[key], (i, key, sr[key], sg[key])
    assert worst <= 1e-4
    rc, _ = rp.export(False)
    gc, _ = gp.volume().export(False)
    key = lambda c: np.lexsort((c[:, 2], c[:, 1], c[:, 0]))  # noqa: E731
    assert rc.shape == gc.shape and (rc[key(rc)] == gc[key(gc)]).all()
