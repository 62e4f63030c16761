#!/usr/bin/env python
"""NEXT-4 comparator / ablation benches (timing on synthetic data; accuracy is out of scope).

    python tools/bench_modes.py [--out profiles/modes_r2.jsonl]

1. Calibration modes on the LLaVA-NeXT-7B shape (b = 32, 1024 units): the paper's default
   (centered, query-weighted: P:176-186), the uncentered K^T K (north_star's literal wording),
   the query-agnostic K-only PCA (the ablation's "Q-agnostic" arm, tab:rotatek-ablation)
   and W = 0, each with both solvers (Jacobi eigendecomposition, subspace iteration T = 5):
   calibrate / compress / decode time per layer, and -- as a synthetic-data proxy only -- the
   deviation of the r = 32 output from exact attention over the same tokens (our dense mode:
   r = d, R = I), mean and max over query heads of ||o - o_dense||_inf / ||o_dense||_inf.
2. Config 4 (PAPER.md P:26 fig:introduction; north_star): joint token-channel pruning
   (FastV-style 0.30x tokens = 864 survivors + 0.25x Key channels, r = 32) against token-only
   pruning at matched KV bytes (0.20x tokens = 576, dense keys), LLaVA shape, b = 64: decode
   time, algorithmic bytes and achieved bandwidth of each (CUDA graph over distinct layers).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_19218_b200 as rk  # noqa: E402
from workload import CONFIGS, decode_bytes, make_workload  # noqa: E402
from workload.gen import draw_v0  # noqa: E402


def dev(t):
    x = np.ascontiguousarray(t.bits)
    return torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).cuda()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def graph_decode_us(layers, reps=30):
    """us per decode launch: CUDA graph over the given (args, out) layers (each > L2)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for a, kw in layers:
            rk.decode_attn(*a, **kw, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for a, kw in layers:
                rk.decode_attn(*a, **kw, stream=s)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (reps * len(layers))


def modes(out):
    cfg = CONFIGS["llava_b32"]
    w = make_workload(cfg, threads=os.cpu_count() or 8)
    K, V, Qw, q = dev(w["K"]), dev(w["V"]), dev(w["Qw"]), dev(w["q"])
    Kx, Vx = dev(w["Ktext"]), dev(w["Vtext"])
    d = cfg.head_dim
    # exact attention over the same tokens: dense mode (r = d, R = I shared, no bias)
    eye = torch.eye(d, device="cuda").unsqueeze(0).contiguous()
    dense = rk.decode_attn(q, K, V, eye, torch.zeros(1, d, device="cuda"), Kx, Vx)
    V0 = torch.from_numpy(draw_v0(cfg)).cuda()
    flags = {"default": (rk.CENTER | rk.QUERY_WEIGHT, True), "uncentered": (rk.QUERY_WEIGHT, True),
             "q_agnostic": (rk.CENTER, True), "window_0": (rk.CENTER | rk.QUERY_WEIGHT, False)}
    for name, (fl, with_q) in flags.items():
        for solver in ("jacobi", "subspace"):
            if solver == "jacobi":
                cal_fn = lambda: rk.calibrate(K, Qw if with_q else None, cfg.rank, fl)  # noqa: E731
            else:
                cal_fn = lambda: rk.calibrate_subspace(K, Qw if with_q else None, V0, fl)  # noqa: E731
            ms_cal = timed(cal_fn, 3)
            cal = cal_fn()
            us_cmp = 1e3 * timed(lambda: rk.compress_kv(K, cal["R"]), 5)
            Kc = rk.compress_kv(K, cal["R"])
            o = rk.decode_attn(q, Kc, V, cal["R"], cal["dmu"], Kx, Vx)
            us_dec = graph_decode_us([((q, Kc, V, cal["R"], cal["dmu"], Kx, Vx), {"out": torch.empty_like(o)})])
            torch.cuda.synchronize()
            rel = ((o - dense).abs().amax(-1) / dense.abs().amax(-1)).flatten()
            rec = {"bench": "calibration_mode", "config": cfg.name, "mode": name, "solver": solver,
                   "flags": fl, "q_window": cfg.q_window if with_q else 0,
                   "calibrate_ms_per_layer": round(ms_cal, 3), "compress_us_per_layer": round(us_cmp, 1),
                   "decode_us_per_layer_single_layer_graph": round(us_dec, 2),
                   "dev_vs_dense_mean": float(rel.mean()), "dev_vs_dense_max": float(rel.max()),
                   "note": "deviation from exact attention on synthetic data: a proxy, not accuracy"}
            print(json.dumps(rec), flush=True)
            out.write(json.dumps(rec) + "\n")


def joint_vs_tokenonly(out):
    res = {}
    for name in ("joint_b64", "tokenonly_b64"):
        cfg = CONFIGS[name]
        w = make_workload(cfg, threads=os.cpu_count() or 8)
        K, V, Qw, q = dev(w["K"]), dev(w["V"]), dev(w["Qw"]), dev(w["q"])
        Kx, Vx = dev(w["Ktext"]), dev(w["Vtext"])
        d = cfg.head_dim
        if cfg.rank == d:  # token-only: dense keys (r = d, R = I shared, no bias)
            R = torch.eye(d, device="cuda").unsqueeze(0).contiguous()
            dmu = torch.zeros(1, d, device="cuda")
            Kc = K
        else:
            cal = rk.calibrate(K, Qw, cfg.rank)
            R, dmu = cal["R"], cal["dmu"]
            Kc = rk.compress_kv(K, R)
        b = decode_bytes(cfg)
        L = max(2, int(600e6 // b) + 1)
        layers = []
        for l in range(L):
            sh = 7 * l
            roll = lambda x: torch.roll(x, sh, 0).contiguous() if l else x  # noqa: E731
            layers.append(((roll(q), roll(Kc), roll(V), R if R.shape[0] == 1 else roll(R),
                            dmu if dmu.shape[0] == 1 else roll(dmu), roll(Kx), roll(Vx)),
                           {"out": torch.empty(q.shape, dtype=torch.float32, device="cuda")}))
        us = graph_decode_us(layers)
        res[name] = {"bench": "config4_matched_bytes", "config": name, "units": cfg.units, "n_vis": cfg.n_vis,
                     "rank": cfg.rank, "decode_bytes_per_layer": b, "decode_us_per_layer": round(us, 2),
                     "gbs": round(b / (us * 1e-6) / 1e9, 1), "layers_in_graph": L}
        del layers, K, V, Kc
        torch.cuda.empty_cache()
    j, t = res["joint_b64"], res["tokenonly_b64"]
    for r in (j, t):
        r["bytes_ratio_joint_over_tokenonly"] = round(j["decode_bytes_per_layer"] / t["decode_bytes_per_layer"], 4)
        r["time_ratio_joint_over_tokenonly"] = round(j["decode_us_per_layer"] / t["decode_us_per_layer"], 4)
        print(json.dumps(r), flush=True)
        out.write(json.dumps(r) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "modes.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        t0 = time.time()
        modes(f)
        joint_vs_tokenonly(f)
        print(f"# {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
