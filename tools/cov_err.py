#!/usr/bin/env python
"""Eigenvalue / projector error of the tensor-core covariance path vs the fp64 oracle on
planted-gap keys with a mean offset (the fp32-window precision question, SURVEY E-6)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2605_19218_b200 as rk  # noqa: E402
from helpers import to_np64, to_torch  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from workload import CONFIGS, make_workload  # noqa: E402

for mean in (5.0, 20.0):
    for n_vis in (777, 2880):
        cfg = CONFIGS["llava_b1"].with_(h_kv=4, n_vis=n_vis, n_text=0)
        w = make_workload(cfg, dist="gap", mean=mean)
        a = rk.calibrate(to_torch(w["K"]), to_torch(w["Qw"]), cfg.rank)
        torch.cuda.synchronize()
        ref = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
        la = to_np64(a["eigvals"])
        err = (np.abs(np.sort(la, 1) - np.sort(ref["lam"], 1)).max(1) / np.abs(ref["lam"]).max(1)).max()
        Ra = to_np64(a["R"])
        perr = max(np.linalg.norm(Ra[u] @ Ra[u].T - ref["R"][u] @ ref["R"][u].T) for u in range(cfg.units))
        print(f"mean {mean} N {n_vis}: eig err {err:.2e} (gate 2e-5), projector {perr:.2e} (gate 1e-4)")
