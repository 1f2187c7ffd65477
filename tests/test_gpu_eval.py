"""NearestDistances / DistanceCdf on the GPU (rf_eval.cu): the reference's
KATs (test_eval.cpp:115-172, acceptance.cpp:600-616) and bit-exact parity with
the oracle's GridNn restatement on surface-like clouds, host and device
memory, including degenerate grids."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1905_02082_b200 import api as G
from tests import eval_kats

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kat", [eval_kats.kat_nearest_brute_force, eval_kats.kat_nearest_acceptance,
                                 eval_kats.kat_distance_cdf], ids=lambda f: f.__name__)
def test_gpu_eval_kat(kat):
    kat(G)


def surface_clouds(seed, n_ref, n_q):
    """Reference: points on a noisy sphere + plane (a mesh-like 2-manifold);
    queries: a perturbed resample of the same surfaces plus outliers."""
    rng = np.random.default_rng(seed)

    def sample(n, noise):
        k = n // 2
        d = rng.normal(size=(k, 3))
        s = 1.5 * d / np.linalg.norm(d, axis=1, keepdims=True) + [0.3, 1.0, 2.0]
        p = np.c_[rng.uniform(-3, 3, n - k), np.full(n - k, -0.5), rng.uniform(-1, 5, n - k)]
        pts = np.concatenate([s, p]) + rng.normal(scale=noise, size=(n, 3))
        return pts.astype(np.float32)

    ref = sample(n_ref, 0.002)
    q = np.concatenate([sample(n_q - 100, 0.01), rng.uniform(-20, 20, (100, 3))]).astype(np.float32)
    return q, ref


@pytest.mark.parametrize("seed,n_ref,n_q", [(1, 20000, 20000), (2, 200000, 50000)])
def test_nearest_matches_oracle(seed, n_ref, n_q):
    q, ref = surface_clouds(seed, n_ref, n_q)
    want = O.nearest_distances(q, ref)
    got = G.nearest_distances(q, ref)
    np.testing.assert_array_equal(got, want)
    dev = G.nearest_distances(torch.from_numpy(q).cuda(), torch.from_numpy(ref).cuda())
    assert dev.is_cuda and dev.dtype == torch.float64
    np.testing.assert_array_equal(dev.cpu().numpy(), want)
    edges = np.arange(1, 41) * 0.0005
    np.testing.assert_array_equal(G.distance_cdf(got, edges), O.distance_cdf(want, edges))
    np.testing.assert_array_equal(G.distance_cdf(dev, edges), O.distance_cdf(want, edges))


def test_nearest_degenerate_grids():
    rng = np.random.default_rng(7)
    q = rng.uniform(-1, 1, (500, 3)).astype(np.float32)
    one = np.array([[0.25, -0.5, 0.125]], np.float32)  # zero-diagonal box: cell = 1e-6
    np.testing.assert_array_equal(G.nearest_distances(q, one), O.nearest_distances(q, one))
    dup = np.repeat(rng.uniform(-1, 1, (5, 3)).astype(np.float32), 50, axis=0)  # duplicates
    np.testing.assert_array_equal(G.nearest_distances(q, dup), O.nearest_distances(q, dup))
    line = np.c_[np.linspace(-2, 2, 3000), np.zeros(3000), np.zeros(3000)].astype(np.float32)  # flat box
    np.testing.assert_array_equal(G.nearest_distances(q, line), O.nearest_distances(q, line))
    tiny = (rng.uniform(-1, 1, (400, 3)) * 1e-5).astype(np.float32)  # box smaller than 256 * 1e-6
    np.testing.assert_array_equal(G.nearest_distances(q * 1e-5, tiny), O.nearest_distances(q * 1e-5, tiny))


def test_nearest_on_extracted_mesh():
    """The reference's model-accuracy use (tools/main.cpp:341-372): mesh
    vertices of a fused volume against a second extraction's vertices."""
    from tests.test_gpu_parity import frame
    from paper_1905_02082_b200 import scenes
    s = O.Scene(scenes.bench_script(dynamic=False, frames=10, seed=42))
    v = G.TsdfVolume(G.volume_config())
    _, pose = s.camera(0)
    f = s.render(0)
    fr = frame(s.k, f["depth"], f["rgb"])
    v.allocate_for_frame(fr, pose)
    v.integrate(fr, pose)
    xyz = v.extract_mesh(0)[0]
    assert len(xyz) > 10000
    ref = xyz[::3]
    q = xyz + np.float32(0.001)
    np.testing.assert_array_equal(G.nearest_distances(q, ref), O.nearest_distances(q, ref))
