"""Worker for tests/test_replicas.py: the bench's replica harness
(paper_1905_02082_b200/replicas.py) under gloo on CPU. Each rank tracks its
own small synthetic sequence (seed 43 + rank) with the CPU oracle standing in
for the per-GPU pipeline; rank 0 prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch.distributed as dist  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1905_02082_b200 import replicas, scenes  # noqa: E402

STEPS = 3


def main():
    R = replicas.init("gloo")
    seed = replicas.sequence_seed(43, R)
    s = O.Scene(scenes.room_script(with_mover=True, width=64, height=48, frames=STEPS + 1, seed=seed))
    frames = [s.render(i) for i in range(len(s))]
    p = O.Pipeline(O.pipe_cfg(refine=False, volume=O.vol_cfg(voxel_size=0.04, max_blocks=50000)))
    p.process_frame(frames[0]["depth"], frames[0]["rgb"], s.k, 0.0)
    replicas.barrier(R)
    t0 = time.perf_counter()
    for i in range(1, STEPS + 1):
        p.process_frame(frames[i]["depth"], frames[i]["rgb"], s.k, i / 30.0)
    mine = time.perf_counter() - t0
    (sec,) = replicas.max_over_ranks(R, [mine])
    checksum = float(frames[1]["depth"][::7, ::7].sum())
    info = [None] * R.world
    dist.all_gather_object(info, {"rank": R.rank, "seed": seed, "sec": mine, "checksum": checksum})
    if R.lead:
        print(json.dumps({"value": replicas.job_rate(R, STEPS, sec), "max_sec": sec, "world": R.world,
                          "ranks": info}), flush=True)
    replicas.finish(R)


if __name__ == "__main__":
    main()
