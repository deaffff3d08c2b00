"""Multi-GPU plumbing for batches of independent plans.

Plans are independent, so the data path needs no collective: each rank owns
a contiguous shard of the batch and runs its own PlanBatch. torch.distributed
(NCCL on GPUs, gloo on CPU) carries only the control traffic: a barrier
around timed regions, max-over-ranks times, sums of work counters and the
final gather of per-plan summaries.
"""

from __future__ import annotations

import os

import numpy as np


def shard(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) of `total` plans for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def env_rank() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _reduce(x: float, op_name: str, device=None) -> float:
    dist = _dist()
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op_name))
    return float(t.item())


def reduce_max(x: float, device=None) -> float:
    return _reduce(x, "MAX", device)


def reduce_sum(x: float, device=None) -> float:
    return _reduce(x, "SUM", device)


def barrier():
    dist = _dist()
    if dist is not None:
        dist.barrier()


def gather_summaries(summary: dict) -> dict:
    """Concatenate per-rank per-plan arrays (rank order = plan order)."""
    dist = _dist()
    if dist is None:
        return summary
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, {k: np.asarray(v) for k, v in summary.items()})
    return {k: np.concatenate([p[k] for p in parts]) for k in summary}
