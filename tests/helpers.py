"""Test helpers: host <-> torch conversion of generator bytes and the parity metric."""
import numpy as np


def to_torch(t, device="cuda"):
    """workload.Tensor -> torch tensor with the identical bytes."""
    import torch
    if t.dtype == "bf16":
        x = torch.from_numpy(np.ascontiguousarray(t.bits).view(np.int16)).view(torch.bfloat16)
    else:
        x = torch.from_numpy(np.ascontiguousarray(t.bits))
    return x.to(device)


def np_bf16(x_f64):
    """fp64 array holding bf16-exact values -> torch bf16 tensor (exact)."""
    import torch
    return torch.from_numpy(np.asarray(x_f64, dtype=np.float32)).to(torch.bfloat16)


def to_np64(x):
    return x.detach().float().cpu().numpy().astype(np.float64)


def max_rel_err(out, ref):
    """Reading Q23: per output row (u, g) ||o - r||_inf / ||r||_inf, max over rows."""
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    num = np.abs(out - ref).max(axis=-1)
    den = np.abs(ref).max(axis=-1)
    return float((num / den).max())


def mask_bits_u32(mask_i32):
    return np.asarray(mask_i32).astype(np.int64).astype(np.uint32)
