"""One engine per GPU, prefix-affinity groups partitioned across ranks.

The reference places a whole fork group on one engine (scheduler.py:198-221,
`shared-queue` / `shared-ctx` affinity); with one engine per B200 that is
the multi-GPU partition, so the decode path needs no collective.  These
helpers cover the launcher side: which groups a rank owns and the
max-over-ranks timing reduction (the only collective, outside the data path).
"""

from __future__ import annotations

import os
from typing import List, Optional


def world() -> tuple:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def group_owner(group: int, world_size: int) -> int:
    """Rank that hosts fork group `group` (round-robin, whole groups only)."""
    return group % world_size


def rank_groups(rank: int, num_groups: int, world_size: int) -> List[int]:
    return [g for g in range(num_groups) if group_owner(g, world_size) == rank]


def max_over_ranks(value: float, device: Optional[object] = None) -> float:
    """Max of a per-rank scalar (device time) over the process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device: Optional[object] = None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
