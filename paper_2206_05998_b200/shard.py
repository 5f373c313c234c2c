"""Multi-GPU slot sharding: one process per GPU, a static
contiguous partition of independent slots, no collective on the data path.

The only cross-rank traffic is host-side bookkeeping after the device work:
the per-slot results (bit-error counters, status) are gathered to rank 0, and
timings are reduced with MAX (a multi-GPU number is the slowest rank's).
"""
from __future__ import annotations

import numpy as np


def slot_range(total: int, world: int, rank: int):
    """Contiguous block partition: slots [start, stop) of rank `rank`."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad partition arguments")
    start = rank * total // world
    stop = (rank + 1) * total // world
    return start, stop


def slot_seeds(total: int, world: int, rank: int, base: int = 1000) -> np.ndarray:
    """Master seeds (base + global slot index) of this rank's slots."""
    start, stop = slot_range(total, world, rank)
    return np.arange(base + start, base + stop, dtype=np.uint64)


def gather_to_rank0(local: np.ndarray):
    """Concatenate every rank's per-slot rows (in rank = slot order) on rank 0;
    other ranks get None.  Works with any torch.distributed backend."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    parts = [None] * dist.get_world_size() if dist.get_rank() == 0 else None
    dist.gather_object(np.ascontiguousarray(local), parts, dst=0)
    if dist.get_rank() != 0:
        return None
    return np.concatenate(parts, axis=0)


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a scalar over ranks (device timing: the slowest rank)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
