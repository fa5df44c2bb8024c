"""Frame sharding across ranks (one process per GPU).

Frames are independent: each rank segments a contiguous
shard of the batch and nothing crosses GPUs on the data path.  Results are
only gathered when a caller asks for them (to rank 0 by default).  The
reference has no multi-process code; its only concurrency is the thread pool
of ``segment_in_parallel`` (pipeline.py:170-197), whose ordering contract
("output order matches input order") the gather keeps.
"""

from __future__ import annotations

import numpy as np
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced [start, stop) of ``n`` frames for ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def segment_sharded(frames: np.ndarray, segment_fn, group=None, dst: int | None = 0):
    """Segment this rank's shard of ``frames`` with ``segment_fn`` and gather.

    ``segment_fn(shard) -> (labels [n,H,W] int32, n_clusters [n] int32)`` runs
    on the local device (the GPU pipeline in production).  Returns the full
    ``(labels, n_clusters)`` on ``dst`` (all ranks when ``dst is None``) and
    ``None`` elsewhere.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    start, stop = shard_range(frames.shape[0], rank, world)
    labels, ncl = segment_fn(frames[start:stop])
    part = (start, np.asarray(labels), np.asarray(ncl))
    if world == 1:
        return part[1], part[2]
    if dst is None:
        parts = [None] * world
        dist.all_gather_object(parts, part, group=group)
    else:
        parts = [None] * world if rank == dst else None
        dist.gather_object(part, parts, dst=dst, group=group)
        if rank != dst:
            return None
    parts.sort(key=lambda p: p[0])
    return np.concatenate([p[1] for p in parts]), np.concatenate([p[2] for p in parts])
