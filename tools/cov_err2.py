#!/usr/bin/env python
"""Projector / eigenvalue error of the tensor-core vs CUDA-core covariance paths against the
fp64 oracle on the shapes of tests/test_gpu_parity.py::test_calibrate_tensor_core_matches_simt."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2605_19218_b200 as rk  # noqa: E402
from helpers import to_np64, to_torch  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from workload import CONFIGS, make_workload  # noqa: E402

for h_kv, n_vis in ((1, 1), (3, 777), (40, 300), (2, 2048), (4, 4096)):
    cfg = CONFIGS["llava_b1"].with_(h_kv=h_kv, n_vis=n_vis, n_text=0)
    w = make_workload(cfg, dist="gap", mean=5.0)
    K, Qw = to_torch(w["K"]), to_torch(w["Qw"])
    out = {}
    for name, fl in (("tc", rk.DEFAULT_FLAGS), ("simt", rk.DEFAULT_FLAGS | rk.SIMT_ONLY)):
        out[name] = rk.calibrate(K, Qw, cfg.rank, fl)
    torch.cuda.synchronize()
    ref = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    msg = []
    for name, cal in out.items():
        R = to_np64(cal["R"])
        pe = max(np.linalg.norm(R[u] @ R[u].T - ref["R"][u] @ ref["R"][u].T) for u in range(cfg.units))
        le = (np.abs(np.sort(to_np64(cal["eigvals"]), 1) - np.sort(ref["lam"], 1)).max(1) / np.abs(ref["lam"]).max(1)).max()
        msg.append(f"{name}: proj {pe:.3e} eig {le:.2e}")
    print(f"h_kv {h_kv} N {n_vis}: " + "  ".join(msg))
