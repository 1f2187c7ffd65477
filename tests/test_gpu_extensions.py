"""The opt-in extensions (Huber-weighted registration, the free-space mask
term; see test_oracle_extensions.py) on the CUDA path against the oracle's
restatement of them, with the same bars as the reference path: normal
equations within 1e-9, poses within 1e-4, iteration / registration / masked
pixel counts equal, masks bit-exact. Off (the default) they leave the
reference path untouched: that path is what every other parity test runs.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from paper_1905_02082_b200 import scenes
from tests.test_gpu_parity import POSE_TOL_R, POSE_TOL_T, corner, frame, pose_error  # noqa: F401 (fixture)

pytestmark = pytest.mark.gpu

HUBER = dict(huber_depth=0.01, huber_color=0.05)


def test_linearize_huber_matches_oracle(corner):  # noqa: F811
    c = corner
    for cw in (0.0, 0.025):
        o = c["ov"].linearize(c["r"]["depth"], c["r"]["rgb"], c["s"].k, c["init"], O.reg_cfg(color_weight=cw, **HUBER))
        g = c["gv"].linearize(frame(c["s"].k, c["r"]["depth"], c["r"]["rgb"]), c["init"],
                              G.registration_config(color_weight=cw, **HUBER))
        p = c["ov"].linearize(c["r"]["depth"], c["r"]["rgb"], c["s"].k, c["init"], O.reg_cfg(color_weight=cw))
        assert o["valid"] == g["valid"] > 1000
        assert np.abs(o["H"] - p["H"]).max() > 1e-6 * np.abs(p["H"]).max()  # the weights took effect
        np.testing.assert_allclose(g["H"], o["H"], rtol=1e-9, atol=1e-9 * np.abs(o["H"]).max())
        np.testing.assert_allclose(g["b"], o["b"], rtol=1e-9, atol=1e-9 * np.abs(o["b"]).max())
        assert g["error"] == pytest.approx(o["error"], rel=1e-9)


def test_register_huber_matches_oracle(corner):  # noqa: F811
    c = corner
    k = c["s"].k
    o = c["ov"].register(c["r"]["depth"], c["r"]["rgb"], k, c["init"], None, O.reg_cfg(**HUBER))
    g = c["gv"].register(frame(k, c["r"]["depth"], c["r"]["rgb"]), c["init"], None, G.registration_config(**HUBER))
    dt, dr = pose_error(o["pose"], g["pose"])
    assert dt <= POSE_TOL_T and dr <= POSE_TOL_R
    assert g["iterations"] == o["iterations"] and g["converged"] == o["converged"]


def run_pipelines(ocfg, gcfg, n=20):
    s = O.Scene(scenes.room_script(with_mover=True, width=320, height=240, frames=n))
    op = O.Pipeline(ocfg)
    gp = G.Pipeline(gcfg)
    worst, mism = 0.0, 0
    gp.masked = []
    for i in range(n):
        f = s.render(i)
        so, po = op.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])
        sg, pg = gp.process_frame(frame(s.k, f["depth"], f["rgb"], f["timestamp"]))
        worst = max(worst, *pose_error(po, pg))
        gp.masked.append(sg["masked_pixels"])
        mism += sum(so[key] != sg[key] for key in ("registrations", "iterations", "masked_pixels", "tracking_lost"))
        if i > 0 and ocfg.dynamics_enabled:
            om, gm = op.last_mask(s.k), gp.last_mask_image(s.k)
            assert (om is None) == (gm is None) and (om is None or (om == gm).all()), i
            # residuals at the final poses (equal to ~1e-12, not bit for bit): the valid
            # flags, incl. the free-space term's sign bit, agree up to sign flips of ~0 residuals
            (osq, ov), (gsq, gv) = op.last_residuals(s.k), gp.last_residuals(s.k)
            assert (ov != gv).sum() <= 1e-4 * ov.size and np.abs(osq.astype(np.float64) - gsq).max() < 1e-9, i
    return worst, mism, op, gp


@pytest.mark.parametrize("dynamics", [False, True])
def test_pipeline_huber_matches_oracle(dynamics):
    worst, mism, _, _ = run_pipelines(
        O.pipe_cfg(refine=False, dynamics=dynamics, reg=O.reg_cfg(threads=8, **HUBER)),
        G.pipeline_config(refine=False, dynamics=dynamics, registration=G.registration_config(**HUBER)))
    assert worst <= 1e-4 and mism == 0


def test_mask_free_space_bitexact():
    rng = np.random.default_rng(11)
    h, w = 96, 128
    depth = (1.0 + 0.5 * (rng.random((h, w)) < 0.3) + 0.003 * rng.standard_normal((h, w))).astype(np.float32)
    sq = (rng.random((h, w)) * 0.004).astype(np.float32)
    valid = rng.choice(np.array([0, 1, 3], np.uint8), size=(h, w), p=[0.1, 0.45, 0.45])
    sq[30:60, 40:90] = 0.002
    valid[30:60, 40:90] = 3
    for fs in (0.0, 0.02, 0.03):
        oc = O.mask_cfg(free_space=fs)
        gc = G.mask_config(free_space=fs)
        om, gm = O.build_mask(sq, valid, depth, oc), G.build_mask(sq, valid, depth, gc)
        assert (om == gm).all(), fs
        if fs == 0.03:
            assert gm.sum() > G.build_mask(sq, valid, depth, G.mask_config()).sum()


def test_pipeline_free_space_matches_oracle():
    worst, mism, op, gp = run_pipelines(
        O.pipe_cfg(refine=False, reg=O.reg_cfg(threads=8), mask=O.mask_cfg(free_space=0.02)),
        G.pipeline_config(refine=False, mask=G.mask_config(free_space=0.02)))
    assert worst <= 1e-4 and mism == 0
    s = O.Scene(scenes.room_script(with_mover=True, width=320, height=240, frames=20))
    ref = O.Pipeline(O.pipe_cfg(refine=False, reg=O.reg_cfg(threads=8)))
    plain = [ref.process_frame(f["depth"], f["rgb"], s.k, f["timestamp"])[0]["masked_pixels"]
             for f in (s.render(i) for i in range(20))]
    assert gp.masked != plain and sum(gp.masked) > sum(plain)  # the term took effect
