"""Element partitioning across GPUs (one process per GPU) and the max-over-ranks
timing reduction.  Elements are independent, so there is no collective on the
data path; torch.distributed is used only for the barrier
and the timing / checksum reductions outside the fill."""
from __future__ import annotations


def element_range(rank: int, world: int, n_total: int) -> tuple[int, int]:
    """Contiguous strong-scaling partition: GPU g gets [floor(g E / G), floor((g+1) E / G))."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world


def weak_range(rank: int, n_per_rank: int) -> tuple[int, int]:
    """Weak scaling: every rank fills its own n_per_rank elements."""
    return rank * n_per_rank, (rank + 1) * n_per_rank


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
