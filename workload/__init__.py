"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic)."""
from .gen import CONFIGS, Config, Tensor, make_workload, draw_unit, decode_bytes, decode_flops, compress_bytes, f32_to_bf16_bits, bf16_bits_to_f32  # noqa: F401
