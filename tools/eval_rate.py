"""NearestDistances throughput on mesh-sized clouds (the model-accuracy
evaluation, tools/main.cpp:341-372): GPU device-resident, GPU from host
arrays, and the oracle's GridNn on a bounded query sample (1 thread)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1905_02082_b200 import api as G  # noqa: E402
from tests.test_gpu_eval import surface_clouds  # noqa: E402


def main():
    for n in (1_000_000, 4_000_000):
        q, ref = surface_clouds(9, n, n)
        dq, dr = torch.from_numpy(q).cuda(), torch.from_numpy(ref).cuda()
        G.nearest_distances(dq, dr)
        torch.cuda.synchronize()
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            out = G.nearest_distances(dq, dr)
        torch.cuda.synchronize()
        dev_ms = (time.perf_counter() - t0) / reps * 1e3
        t0 = time.perf_counter()
        host = G.nearest_distances(q, ref)
        host_ms = (time.perf_counter() - t0) * 1e3
        sample = 20000
        t0 = time.perf_counter()
        want = O.nearest_distances(q[:sample], ref)
        o_s = time.perf_counter() - t0
        assert np.array_equal(want, host[:sample]) and np.array_equal(out[:sample].cpu().numpy(), want)
        print(f"n={n}: gpu device {dev_ms:.2f} ms ({n / dev_ms / 1e3:.1f} Mq/s), gpu from host {host_ms:.1f} ms, "
              f"oracle (incl. grid build) {o_s:.2f} s for {sample} queries")


if __name__ == "__main__":
    main()
