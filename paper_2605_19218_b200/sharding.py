"""Host-side partitioning of RotateK units across ranks (one process per GPU).

Every hot-path step is independent per unit u = b * H_kv + h_kv, so a
rank's share of a batch is a contiguous unit range, i.e. a pointer offset into the
[U, ...] tensors -- no collective on the data path.

* weak scaling (bench default): every rank owns a full per-GPU batch; rank r's units are
  the global units [r*U, (r+1)*U).
* strong scaling: a fixed global batch of U units is split into contiguous ranges of
  ceil(U / world) (the last rank may get fewer, ranks beyond U get none).
* token sharding (U < world, e.g. Qwen b1 with 4 units on 8 GPUs): every
  rank holds all units but only its contiguous slice of the visual (and text) tokens; it
  runs Alg. 2 over its slice (rotatek_decode_attn_partial), the [U, G, d+2] states are
  all-gathered (the one collective: NCCL all_gather_into_tensor) and merged
  (rotatek_merge_partials) -- the exact online-softmax merge of App. C.
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


def token_slice(n: int, world: int, rank: int) -> range:
    """Balanced contiguous slice of n tokens for `rank` (sizes differ by at most one)."""
    return range(n * rank // world, n * (rank + 1) // world)


def _all_gather(out, inp, group=None):
    """all_gather_into_tensor(out, inp): NCCL over NVLink for device tensors; with a gloo
    group (CPU tests, or several ranks sharing one GPU) the device rows are staged through
    the host -- the collective only, the hot path stays in the CUDA kernels."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl" or not inp.is_cuda:
        dist.all_gather_into_tensor(out, inp, group=group)
        return out
    host = torch.empty(out.shape, dtype=out.dtype)
    dist.all_gather_into_tensor(host, inp.cpu(), group=group)
    out.copy_(host)
    return out


def decode_unit_sharded(q, K_comp, V, R, dmu, K_text=None, V_text=None, scale=0.0, group=None,
                        total_units=None):
    """Strong scaling by unit ranges: this rank holds the units
    strong_units(total_units, rank, world) of a global batch (its tensors are those rows),
    decodes them, and the outputs are gathered -- the one NCCL all_gather_into_tensor of
    out [U, G, d] fp32 (north_star: "NCCL over NVLink is used only to gather outputs").
    Returns the full [total_units, G, d] output on every rank."""
    import torch
    import torch.distributed as dist

    from . import rotatek as rk
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n_local = q.shape[0]
    out = rk.decode_attn(q, K_comp, V, R, dmu, K_text, V_text, scale) if n_local else \
        torch.empty((0,) + tuple(q.shape[1:]), dtype=torch.float32, device=q.device)
    if world == 1:
        return out
    total = total_units if total_units is not None else n_local * world
    per = -(-total // world)
    send = torch.zeros((per,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    send[:n_local] = out
    full = torch.empty((world * per,) + tuple(out.shape[1:]), dtype=out.dtype, device=out.device)
    _all_gather(full, send, group)
    return full[:total]


def decode_token_sharded(q, K_comp, V, R, dmu, K_text=None, V_text=None, scale=0.0, group=None):
    """Token-sharded Alg. 2: this rank's cache shard -> the full output [U, G, d] on every
    rank.  One all-gather of the [U, G, d+2] fp32 states, then the merge kernel."""
    import torch
    import torch.distributed as dist

    from . import rotatek as rk
    part = rk.decode_attn_partial(q, K_comp, V, R, dmu, K_text, V_text, scale)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return rk.merge_partials(part[None])
    parts = torch.empty((world * part.shape[0],) + tuple(part.shape[1:]), dtype=part.dtype,
                        device=part.device)
    _all_gather(parts, part, group)
    return rk.merge_partials(parts.view((world,) + tuple(part.shape)))
