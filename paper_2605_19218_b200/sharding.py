"""Host-side partitioning of RotateK units across ranks (one process per GPU).

Every hot-path step is independent per unit u = b * H_kv + h_kv, so a
rank's share of a batch is a contiguous unit range, i.e. a pointer offset into the
[U, ...] tensors -- no collective on the data path.

* weak scaling (bench default): every rank owns a full per-GPU batch; rank r's units are
  the global units [r*U, (r+1)*U).
* strong scaling: a fixed global batch of U units is split into contiguous ranges of
  ceil(U / world) (the last rank may get fewer, ranks beyond U get none).
"""
from __future__ import annotations


def weak_units(units_per_rank: int, rank: int) -> range:
    return range(rank * units_per_rank, (rank + 1) * units_per_rank)


def strong_units(total_units: int, rank: int, world: int) -> range:
    per = -(-total_units // world)
    lo = min(total_units, rank * per)
    hi = min(total_units, lo + per)
    return range(lo, hi)


def max_over_ranks(value: float, group=None) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
