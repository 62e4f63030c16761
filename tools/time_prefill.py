#!/usr/bin/env python
"""Prefill kernel timings (experiments): compress (K -> K~) and the covariance pass
(rotatek_calib_accumulate = sigma + covariance + state add) on random bf16 keys, CUDA
events, several distinct key buffers so nothing is L2-resident."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_19218_b200 as rk  # noqa: E402
from workload import CONFIGS  # noqa: E402


def t(fn, n, reps=10):
    for i in range(2):
        fn(i % n)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n):
            fn(i)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / n)
    ts.sort()
    return ts[len(ts) // 2]


for name in sys.argv[1:] or ["llava_b32", "qwen_b32_r32", "long_b16"]:
    cfg = CONFIGS[name]
    U, N, d, r = cfg.units, cfg.n_vis, cfg.head_dim, cfg.rank
    n = 3
    Ks = [torch.randn(U, N, d, device="cuda").bfloat16() for _ in range(n)]
    Qw = torch.randn(U, cfg.group, 32, d, device="cuda").bfloat16()
    R = torch.linalg.qr(torch.randn(U, d, d, device="cuda"))[0][:, :, :r].contiguous()
    out = torch.empty(U, N, r, device="cuda").bfloat16()
    st = rk.calib_state(U, d)
    kb = U * N * d * 2
    tc = t(lambda i: rk.compress_kv(Ks[i], R, out=out), n)
    tcov = t(lambda i: rk.calib_accumulate(Ks[i], Qw, st), n)
    print(f"{name}: compress {tc:.1f} us ({(kb + U * N * r * 2) / tc / 1e3:.0f} GB/s)   "
          f"covariance+accumulate {tcov:.1f} us ({kb / tcov / 1e3:.0f} GB/s of K)", flush=True)
