"""Seeded synthetic workloads for the RotateK hot path.

This module is shared by the oracle side (tests, cpu_baseline) and the CUDA
side (tests, bench).  It holds NONE of the method's arithmetic: it only draws
random numbers, shapes them like the paper's workloads and rounds them to the
cache dtype (RNE), so that both sides consume identical bytes.

Recipe:
  * Every unit u (= batch element b * H_kv + kv head) has its own generator
    ``numpy.random.default_rng([seed, u])`` (PCG64), so any unit can be
    regenerated alone (sampled full-size parity) and the bytes do not depend
    on chunking or thread count.  seed = 1000 * config_id + layer.
  * ``nat`` (natural; mimics fig:motivation P:47-62: a few outlier channels and
    RoPE token dependence): K_pre = kappa * Z A^T / sqrt(d) + 0.3 E + 0.5 with
    Z, E ~ N(0,1) [tokens, d], A ~ N(0,1) [d, d] with row i scaled by
    exp(-i/12); channels round(40 d/128) and round(100 d/128) scaled x8; then
    RoPE (base 10000, rotate-half pairs (i, i + d/2)) at positions 0..N+M-1.
    Visual keys take positions 0..N-1, text keys N..N+M-1.  V ~ N(0,1).
    Q_W rows and q ~ N(0,1) with a per-unit random 20% of channels x4.
  * ``gap`` (planted spectral gap, for calibration parity): K = (Z diag(s)) Q^T
    + mean with Q random orthogonal, s = linspace(3, 1, r) ++ 0.05 * 1_{d-r};
    queries scaled by ``logit_scale``.
  * Token-pruned caches (config "joint"): the full 2880-position cache is drawn
    and a seeded sorted random subset of round(0.30 * 2880) = 864 positions is
    kept (FastV-like scattered survivors keep their RoPE phases).
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field, replace

import numpy as np


# --------------------------------------------------------------------------
# configurations (BASELINE.json "configs")
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    config_id: int
    batch: int
    h_kv: int
    group: int          # G = H_q / H_kv
    head_dim: int       # d
    rank: int           # r kept rotated channels
    n_vis: int          # N visual tokens per unit (after token pruning)
    n_text: int         # M full-d prompt/text tokens per unit
    q_window: int = 32  # W
    dtype: str = "bf16"
    layers: int = 1     # model layers (LLaVA 32, Qwen 28) -- bench times a subset
    dist: str = "nat"
    n_vis_full: int = 0  # >0: draw this many positions and keep a sorted subset of n_vis
    extra: dict = field(default_factory=dict, compare=False)

    @property
    def units(self) -> int:
        return self.batch * self.h_kv

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: toy (oracle finishes in milliseconds); 8 decode steps grow M 0 -> 8
    "toy": Config("toy", 0, batch=1, h_kv=1, group=1, head_dim=16, rank=4, n_vis=64,
                  n_text=0, q_window=32),
    # configs[1]: LLaVA-NeXT-7B shape (32 MHA heads), 2880 visual + 128 text, 0.25x channels
    "llava_b1": Config("llava_b1", 1, 1, 32, 1, 128, 32, 2880, 128, layers=32),
    "llava_b8": Config("llava_b8", 1, 8, 32, 1, 128, 32, 2880, 128, layers=32),
    "llava_b32": Config("llava_b32", 1, 32, 32, 1, 128, 32, 2880, 128, layers=32),
    # configs[2]: Qwen2.5-VL-7B shape (28 q / 4 kv heads), 4k visual tokens, 0.25x / 0.5x
    "qwen_b1_r32": Config("qwen_b1_r32", 2, 1, 4, 7, 128, 32, 4096, 128, layers=28),
    "qwen_b8_r32": Config("qwen_b8_r32", 2, 8, 4, 7, 128, 32, 4096, 128, layers=28),
    "qwen_b32_r32": Config("qwen_b32_r32", 2, 32, 4, 7, 128, 32, 4096, 128, layers=28),
    "qwen_b32_r64": Config("qwen_b32_r64", 2, 32, 4, 7, 128, 64, 4096, 128, layers=28),
    # configs[3]: joint FastV 0.30x tokens + 0.25x channels, LLaVA shape, batch 64
    "joint_b64": Config("joint_b64", 3, 64, 32, 1, 128, 32, 864, 128, layers=32,
                        n_vis_full=2880),
    # its matched-bytes comparator: token-only 0.20x (576 tokens), dense keys (r = d)
    "tokenonly_b64": Config("tokenonly_b64", 3, 64, 32, 1, 128, 128, 576, 128, layers=32,
                            n_vis_full=2880),
    # configs[4]: long multi-image/video, Qwen shape, 32k visual, batch 16
    "long_b16": Config("long_b16", 4, 16, 4, 7, 128, 32, 32768, 128, layers=28),
}


# --------------------------------------------------------------------------
# dtype helpers (input synthesis: RNE rounding of drawn values to the cache dtype)
# --------------------------------------------------------------------------
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """RNE float32 -> bfloat16, returned as uint16 bit patterns (finite inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    bias = ((b >> 16) & 1) + np.uint32(0x7FFF)
    return ((b + bias) >> 16).astype(np.uint16)


def bf16_bits_to_f32(u: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(u, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


class Tensor:
    """Host array in the cache dtype: ``bits`` (uint16 for bf16, float32 for
    f32) plus an exact float32/float64 view ``values``."""

    def __init__(self, arr: np.ndarray, dtype: str):
        self.dtype = dtype
        if dtype == "bf16":
            self.bits = f32_to_bf16_bits(arr)
        elif dtype == "f32":
            self.bits = np.ascontiguousarray(arr, dtype=np.float32)
        else:
            raise ValueError(dtype)

    @property
    def shape(self):
        return self.bits.shape

    def f32(self) -> np.ndarray:
        return bf16_bits_to_f32(self.bits) if self.dtype == "bf16" else self.bits

    def f64(self) -> np.ndarray:
        return self.f32().astype(np.float64)

    def nbytes(self) -> int:
        return self.bits.nbytes


# --------------------------------------------------------------------------
# per-unit drawing
# --------------------------------------------------------------------------
def _rope(x: np.ndarray, pos: np.ndarray, base: float = 10000.0) -> np.ndarray:
    """Rotary embedding, rotate-half convention, pairs (i, i + d/2)."""
    d = x.shape[-1]
    h = d // 2
    inv = base ** (-np.arange(h, dtype=np.float64) * 2.0 / d)
    ang = pos[:, None].astype(np.float64) * inv[None, :]
    c = np.cos(ang).astype(np.float32)
    s = np.sin(ang).astype(np.float32)
    a, b = x[:, :h], x[:, h:]
    return np.concatenate([a * c - b * s, a * s + b * c], axis=1)


def _outlier_channels(d: int):
    return sorted({min(d - 1, round(40 * d / 128)), min(d - 1, round(100 * d / 128))})


def draw_unit(cfg: Config, seed: int, u: int, dist: str | None = None, *, mean: float = 0.5,
              logit_scale: float = 1.0, kappa: float = 3.0) -> dict:
    """All inputs of one unit as float32 arrays (before dtype rounding)."""
    dist = dist or cfg.dist
    rng = np.random.default_rng([int(seed), int(u)])
    d, r, G, W, M = cfg.head_dim, cfg.rank, cfg.group, cfg.q_window, cfg.n_text
    n_draw = cfg.n_vis_full if cfg.n_vis_full else cfg.n_vis
    T = n_draw + M
    if dist == "nat":
        A = rng.standard_normal((d, d), dtype=np.float32)
        A *= np.exp(-np.arange(d, dtype=np.float32) / 12.0)[:, None]
        Z = rng.standard_normal((T, d), dtype=np.float32)
        E = rng.standard_normal((T, d), dtype=np.float32)
        Kall = (kappa / math.sqrt(d)) * (Z @ A.T) + 0.3 * E + mean
        for ch in _outlier_channels(d):
            Kall[:, ch] *= 8.0
        Kall = _rope(Kall, np.arange(T))
    elif dist == "gap":
        Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
        s = np.concatenate([np.linspace(3.0, 1.0, r), np.full(d - r, 0.05)])
        Z = rng.standard_normal((T, d))
        Kall = ((Z * s[None, :]) @ Q.T + mean).astype(np.float32)
    else:
        raise ValueError(dist)
    if cfg.n_vis_full:
        keep = np.sort(rng.choice(n_draw, size=cfg.n_vis, replace=False))
        Kvis = Kall[keep]
    else:
        Kvis = Kall[:n_draw]
    Ktext = Kall[n_draw:]
    boost = np.ones(d, dtype=np.float32)
    boost[rng.choice(d, size=max(1, round(0.2 * d)), replace=False)] = 4.0
    V = rng.standard_normal((cfg.n_vis, d), dtype=np.float32)
    Vtext = rng.standard_normal((M, d), dtype=np.float32)
    Qw = rng.standard_normal((G, W, d), dtype=np.float32) * boost
    q = rng.standard_normal((G, d), dtype=np.float32) * boost * logit_scale
    return dict(K=Kvis, V=V, Ktext=Ktext, Vtext=Vtext, Qw=Qw, q=q)


def make_workload(cfg: Config, seed: int | None = None, layer: int = 0, units=None,
                  dist: str | None = None, threads: int = 8, **kw) -> dict:
    """Inputs for ``units`` (default: all cfg.units) as ``Tensor`` objects in
    cfg.dtype: K [U,N,d], V [U,N,d], Ktext/Vtext [U,M,d], Qw [U,G,W,d], q [U,G,d]."""
    if seed is None:
        seed = 1000 * cfg.config_id + layer
    ulist = list(range(cfg.units)) if units is None else [int(x) for x in units]
    U = len(ulist)
    d, G, W, M, N = cfg.head_dim, cfg.group, cfg.q_window, cfg.n_text, cfg.n_vis
    bufs = dict(K=np.empty((U, N, d), np.float32), V=np.empty((U, N, d), np.float32),
                Ktext=np.empty((U, M, d), np.float32), Vtext=np.empty((U, M, d), np.float32),
                Qw=np.empty((U, G, W, d), np.float32), q=np.empty((U, G, d), np.float32))

    def one(i):
        x = draw_unit(cfg, seed, ulist[i], dist, **kw)
        for k, v in x.items():
            bufs[k][i] = v

    if U > 4 and threads > 1:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(U)))
    else:
        for i in range(U):
            one(i)
    out = {k: Tensor(v, cfg.dtype) for k, v in bufs.items()}
    out["units"] = np.array(ulist, dtype=np.int64)
    out["seed"] = seed
    return out


def draw_v0(cfg: Config, seed: int | None = None, units=None) -> np.ndarray:
    """Start basis of the subspace iteration ("Sample V with i.i.d. N(0,1) entries", Alg. 1
    l.6): float32 [U, d, r], one generator per unit (stream 1 of default_rng([seed, u, 1]))."""
    if seed is None:
        seed = 1000 * cfg.config_id
    ulist = list(range(cfg.units)) if units is None else [int(x) for x in units]
    out = np.empty((len(ulist), cfg.head_dim, cfg.rank), np.float32)
    for i, u in enumerate(ulist):
        out[i] = np.random.default_rng([int(seed), int(u), 1]).standard_normal(
            (cfg.head_dim, cfg.rank), dtype=np.float32)
    return out


def decode_bytes(cfg: Config) -> int:
    """Algorithmic bytes one decode launch must move:
    K~ U*N*r*s + V U*N*d*s + text 2*U*M*d*s + R_r U*d*r*4 + dmu U*d*4
    + q U*G*d*s + out U*G*d*4."""
    s = 2 if cfg.dtype == "bf16" else 4
    U, N, M, d, r, G = cfg.units, cfg.n_vis, cfg.n_text, cfg.head_dim, cfg.rank, cfg.group
    return (U * N * r * s + U * N * d * s + 2 * U * M * d * s + U * d * r * 4 + U * d * 4
            + U * G * d * s + U * G * d * 4)


def decode_flops(cfg: Config) -> int:
    """Algorithmic flops of one decode launch: q~ (2dr) + bias (2d) per head,
    visual scores 2r + PV 2d per token per head, text 4d per token per head."""
    U, N, M, d, r, G = cfg.units, cfg.n_vis, cfg.n_text, cfg.head_dim, cfg.rank, cfg.group
    return U * G * (2 * d * r + 2 * d + N * (2 * r + 2 * d) + M * 4 * d)


def compress_bytes(cfg: Config) -> int:
    """Algorithmic bytes of calibrate + compress (one pass over K, write K~,
    read Q_W, write R_r and dmu)."""
    s = 2 if cfg.dtype == "bf16" else 4
    U, N, d, r, G, W = cfg.units, cfg.n_vis, cfg.head_dim, cfg.rank, cfg.group, cfg.q_window
    return U * N * d * s + U * N * r * s + U * G * W * d * s + U * d * r * 4 + U * d * 4
