"""Multi-GPU = replicas only.

Exact parity forbids sharding one system: natural-order Gauss-Seidel, ILU(0)
and the Ruge-Stueben first pass each carry a global dependency chain across
any row partition.  Independent systems (Peclet points, method
pairs, Newton steps) are distributed one process per GPU with no collective on
the data path; the only collectives are the timing max and the work sum.
"""
from __future__ import annotations


def assign(n_systems: int, rank: int, world: int) -> list[int]:
    """Round-robin system ids owned by `rank`."""
    return list(range(rank, n_systems, world))


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def reduce_max(x: float, device=None) -> float:
    """Max over ranks (timings: the job ends when the slowest rank ends)."""
    dist = _dist()
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, device=None) -> float:
    dist = _dist()
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def whole_job_throughput(local_units: float, local_seconds: float, device=None) -> float:
    """Units processed by all ranks / the slowest rank's time."""
    return reduce_sum(local_units, device) / reduce_max(local_seconds, device)
