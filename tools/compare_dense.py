#!/usr/bin/env python
"""NEXT-4 comparator: dense decode attention over the same tokens.

The paper's efficiency figure (fig:efficiency) compares RotateK's sparse-channel decode with
a dense FlashAttention decode over the full-d cache.  Here, on B200, for one shape:
  * FlashInfer BatchDecodeWithPagedKVCacheWrapper (library kernel; HND layout, one page of
    N+M tokens per batch element == our [B, H_kv, L, d] layout), dense bf16 K/V;
  * librotatek in dense mode: r = d = 128, one shared R = I (r_units = 1), dmu = 0 --
    i.e. standard attention through our own kernel (validated against FlashInfer);
  * librotatek RotateK decode: r = 32 visual channels + M full-d text tokens (the method).
Random bf16 caches made on the device; L distinct layers per timing loop (each > L2),
back-to-back launches, CUDA events; median µs per layer.

    python tools/compare_dense.py [llava_b32|qwen_b32_r32 ...]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_19218_b200 as rk  # noqa: E402
from workload import CONFIGS, decode_bytes  # noqa: E402


def timeit(fn, layers, reps=20):
    for i in range(3):
        fn(i % layers)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(layers):
            fn(i)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / layers)
    ts.sort()
    return ts[len(ts) // 2]


def run(name):
    import flashinfer
    cfg = CONFIGS[name]
    B, H, G, d, N, M, r = cfg.batch, cfg.h_kv, cfg.group, cfg.head_dim, cfg.n_vis, cfg.n_text, cfg.rank
    U, L = B * H, N + M
    dev = "cuda"
    dense_bytes = 2 * U * L * d * 2 + U * G * d * 2 + U * G * d * 2
    layers = max(2, int(2.5e9 // dense_bytes) + 1)
    layers = min(layers, 6)
    res = {"config": name, "B": B, "H_kv": H, "G": G, "N": N, "M": M, "r": r, "layers": layers}

    # ---- dense caches (shared by FlashInfer and our dense mode)
    Kd = [torch.randn(U, L, d, device=dev).bfloat16() for _ in range(layers)]
    Vd = [torch.randn(U, L, d, device=dev).bfloat16() for _ in range(layers)]
    q = [torch.randn(U, G, d, device=dev).bfloat16() for _ in range(layers)]
    fws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ar = torch.arange(B + 1, dtype=torch.int32, device=dev)
    pages = torch.arange(B, dtype=torch.int32, device=dev)
    last = torch.full((B,), L, dtype=torch.int32, device=dev)
    if G in (1, 2, 4, 8):
        # FlashInfer's decode kernel (group sizes 1/2/4/8 only)
        wrapper = flashinfer.BatchDecodeWithPagedKVCacheWrapper(fws, kv_layout="HND")
        wrapper.plan(ar, pages, last, num_qo_heads=H * G, num_kv_heads=H, head_dim=d, page_size=L,
                     pos_encoding_mode="NONE", q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        res["flashinfer_kernel"] = "BatchDecodeWithPagedKVCacheWrapper"
    else:
        # G = 7 (Qwen2.5-VL): the decode kernel rejects group size 7; the paged prefill
        # kernel with one query token per request computes the same attention
        wrapper = flashinfer.BatchPrefillWithPagedKVCacheWrapper(fws, kv_layout="HND")
        wrapper.plan(ar, ar, pages, last, num_qo_heads=H * G, num_kv_heads=H, head_dim_qk=d,
                     page_size=L, causal=False, pos_encoding_mode="NONE",
                     q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        res["flashinfer_kernel"] = "BatchPrefillWithPagedKVCacheWrapper (qo_len = 1)"
    fo = [None] * layers

    def fi(i):
        fo[i] = wrapper.run(q[i].view(B, H * G, d), (Kd[i].view(B, H, L, d), Vd[i].view(B, H, L, d)))
    t_fi = timeit(fi, layers)

    # ---- ours, dense mode: r = d, R = I shared by every unit, dmu = 0
    eye = torch.eye(d, device=dev).unsqueeze(0).contiguous()
    z = torch.zeros(1, d, device=dev)
    oo = [torch.empty(U, G, d, device=dev) for _ in range(layers)]
    wsd = rk.workspace(rk.make_dims(U, G, d, d, L, 0), rk.OP_DECODE, dev)

    def ours_dense(i):
        rk.decode_attn(q[i], Kd[i], Vd[i], eye, z, out=oo[i], ws=wsd)
    t_od = timeit(ours_dense, layers)
    fi(0)
    ours_dense(0)
    torch.cuda.synchronize()
    ref = fo[0].float().view(U, G, d)
    err = ((oo[0] - ref).abs().amax(-1) / ref.abs().amax(-1)).max().item()

    # ---- ours, RotateK: r visual channels + M full-d text tokens
    del Kd, Vd
    torch.cuda.empty_cache()
    Kc = [torch.randn(U, N, r, device=dev).bfloat16() for _ in range(layers)]
    Vv = [torch.randn(U, N, d, device=dev).bfloat16() for _ in range(layers)]
    Kx = [torch.randn(U, M, d, device=dev).bfloat16() for _ in range(layers)]
    Vx = [torch.randn(U, M, d, device=dev).bfloat16() for _ in range(layers)]
    R = [torch.linalg.qr(torch.randn(U, d, d, device=dev))[0][:, :, :r].contiguous() for _ in range(layers)]
    dm = [torch.randn(U, d, device=dev) * 0.1 for _ in range(layers)]
    wsr = rk.workspace(rk.make_dims(U, G, d, r, N, M), rk.OP_DECODE, dev)

    def ours_rk(i):
        rk.decode_attn(q[i], Kc[i], Vv[i], R[i], dm[i], Kx[i], Vx[i], out=oo[i], ws=wsr)
    t_rk = timeit(ours_rk, layers)

    res.update({
        "flashinfer_dense_us": round(t_fi, 2), "flashinfer_dense_gbs": round(dense_bytes / t_fi / 1e3, 1),
        "ours_dense_us": round(t_od, 2), "ours_dense_gbs": round(dense_bytes / t_od / 1e3, 1),
        "ours_dense_vs_flashinfer_max_rel_err": err,
        "rotatek_us": round(t_rk, 2), "rotatek_gbs": round(decode_bytes(cfg) / t_rk / 1e3, 1),
        "speedup_rotatek_vs_flashinfer_dense": round(t_fi / t_rk, 3),
        "dense_bytes": dense_bytes, "rotatek_bytes": decode_bytes(cfg),
        "timing": "back-to-back launches over distinct layer caches, CUDA events, median",
    })
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["llava_b32", "qwen_b32_r32"]:
        run(n)
