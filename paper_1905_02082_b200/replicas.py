"""Multi-GPU = replicas: one process per GPU, each running an
independent sequence; torch.distributed is used only for the start barrier
and the max-over-ranks of the timings, never on the data path (a frame's pose
depends on the volume after the previous frame, pipeline.cpp:81-115, so a
sequence does not shard).

The same helpers run under gloo on CPU (tests/test_replicas.py) and NCCL on
GPUs (bench.py under torchrun)."""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class Rank:
    rank: int
    world: int
    local: int
    backend: str | None = None

    @property
    def lead(self) -> bool:
        return self.rank == 0


def env() -> Rank:
    return Rank(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None) -> Rank:
    """Joins the process group when WORLD_SIZE > 1 (MASTER_ADDR/PORT from the
    launcher); backend defaults to nccl with CUDA, gloo without."""
    r = env()
    if r.world > 1:
        import torch
        import torch.distributed as dist

        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {"device_id": torch.device("cuda", r.local)} if backend == "nccl" else {}
        dist.init_process_group(backend, **kw)
        r.backend = backend
    return r


def sequence_seed(base: int, r: Rank) -> int:
    """Each replica tracks its own sequence (C5: seeds 43..50)."""
    return base + r.rank


def barrier(r: Rank) -> None:
    if r.world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(r: Rank, values):
    """Element-wise max of per-rank timings (the slowest replica bounds the
    whole-job time)."""
    vals = [float(v) for v in values]
    if r.world == 1:
        return vals
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", r.local) if r.backend == "nccl" else torch.device("cpu")
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def job_rate(r: Rank, units_per_rank: int, seconds_max: float) -> float:
    """Whole-job throughput: units all ranks processed / the slowest rank's time."""
    return r.world * units_per_rank / seconds_max


def finish(r: Rank) -> None:
    if r.world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
