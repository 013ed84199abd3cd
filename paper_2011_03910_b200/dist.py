"""Multi-GPU plumbing: streams sharded over ranks, one final metrics gather.

Streams are independent tracker instances: there is
no exchange step on the hot path, so every rank runs the single-GPU path on
its own contiguous block of streams and the only collective is one
``all_gather`` of a small per-rank metrics tensor at the end (NCCL on GPUs,
gloo in the CPU tests).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

METRIC_FIELDS = ("frames", "ids_issued", "live_tracks", "candidates", "detections", "records", "elapsed_ms")


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    stream_begin: int
    n_streams: int


def env() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def shard_streams(total_streams: int, world: int, rank: int) -> Shard:
    """Contiguous block of streams for ``rank``; the first ``total % world``
    ranks take one extra stream (64 per GPU for config 4 at 8 GPUs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    if total_streams < 0:
        raise ValueError("negative stream count")
    base, extra = divmod(total_streams, world)
    begin = rank * base + min(rank, extra)
    return Shard(rank, world, begin, base + (1 if rank < extra else 0))


def gather_metrics(metrics: dict, device=None):
    """All-gather per-rank metrics (the run's only collective). Returns a list
    of dicts, one per rank, on every rank; works without a process group."""
    import torch

    vals = torch.tensor([float(metrics.get(k, 0.0)) for k in METRIC_FIELDS], dtype=torch.float64,
                        device=device)
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return [dict(zip(METRIC_FIELDS, vals.tolist()))]
    out = [torch.zeros_like(vals) for _ in range(dist.get_world_size())]
    dist.all_gather(out, vals)
    return [dict(zip(METRIC_FIELDS, t.tolist())) for t in out]


def summarize(per_rank: list[dict]) -> dict:
    """Whole-job throughput: frames of all ranks over the slowest rank's time."""
    frames = sum(m["frames"] for m in per_rank)
    slowest = max(m["elapsed_ms"] for m in per_rank) if per_rank else 0.0
    return {"frames": frames, "max_elapsed_ms": slowest,
            "frames_per_s": frames / (slowest / 1e3) if slowest > 0 else 0.0,
            "ids_issued": sum(m["ids_issued"] for m in per_rank),
            "ranks": len(per_rank)}
