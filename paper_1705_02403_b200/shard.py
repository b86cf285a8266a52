"""Multi-GPU plumbing for batched queries.

Independent planning queries shard naturally: rank r of W solves the
contiguous query range `shard_range(...)` on its own GPU with no per-query
communication, and one fixed-size record per query is gathered to rank 0 at
the end (the only collective: torch.distributed over NCCL on the GPU box,
gloo in the CPU tests).  A single query is never split across GPUs
("replicas only" for latency).
"""
from __future__ import annotations

import numpy as np

# One record per query: status, cost, iterations, checks, path_len, num_stats.
RECORD_FIELDS = ("status", "cost", "iterations", "total_collision_checks", "path_len", "num_stats")


def shard_range(total: int, world: int, rank: int) -> range:
    """Contiguous, balanced block of [0, total) for `rank` (sizes differ by
    at most one; earlier ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def weak_range(per_rank: int, rank: int) -> range:
    """Weak scaling: every rank owns `per_rank` queries of its own."""
    return range(rank * per_rank, (rank + 1) * per_rank)


def records(summaries) -> np.ndarray:
    """PlanSummary list -> float64 [count, 6] records (exact for every field:
    counts stay far below 2^53)."""
    return np.array([[getattr(s, f) for f in RECORD_FIELDS] for s in summaries],
                    np.float64).reshape(-1, len(RECORD_FIELDS))


def gather_records(local: np.ndarray, device=None) -> np.ndarray | None:
    """Gather every rank's [count_r, 6] records to rank 0 in rank order.
    Counts may differ per rank (shard_range).  Returns the concatenation on
    rank 0 and None elsewhere; without an initialised process group it
    returns `local`."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cpu") if device is None else torch.device(device)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    width = local.shape[1]
    cap = max(counts)
    buf = torch.zeros((cap, width), dtype=torch.float64, device=dev)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(dev)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    if rank != 0:
        return None
    return np.concatenate([p[:c].cpu().numpy() for p, c in zip(parts, counts)], axis=0)
