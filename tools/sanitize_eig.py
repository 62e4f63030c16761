"""compute-sanitizer target for the r2 eigensolver and covariance changes: the one-sided
Jacobi (hestenes_kernel) with its null-column fallback, rank-deficient C_q, the DMMA
refinement for KC = 40 / 72 and the full refinement (r > 64), and cov_tc with more
(unit, part) items than SMs (persistent CTAs walking several items)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_19218_b200 as rk
from workload import CONFIGS, make_workload


def dev(t):
    return torch.from_numpy(np.ascontiguousarray(t.bits).view(np.int16)).view(torch.bfloat16).cuda()


cases = [("null", CONFIGS["llava_b1"].with_(h_kv=3, n_vis=300, n_text=0), "gap"),
         ("rankdef", CONFIGS["llava_b1"].with_(h_kv=2, n_vis=40, n_text=0), "gap"),
         ("r64", CONFIGS["qwen_b1_r32"].with_(h_kv=2, rank=64, n_vis=260, n_text=0), None),
         ("r100", CONFIGS["llava_b1"].with_(h_kv=2, rank=100, n_vis=260, n_text=0), None),
         ("items>SMs", CONFIGS["llava_b1"].with_(h_kv=160, n_vis=300, n_text=0), None)]
for name, cfg, dist in cases:
    w = make_workload(cfg, dist=dist) if dist else make_workload(cfg)
    K = dev(w["K"])
    if name == "null":
        K[1, :, 7] = 1.25
        K[2, :, 3] = 0.0
    for fl in (rk.DEFAULT_FLAGS, rk.DEFAULT_FLAGS | rk.EIG_TWOSIDED):
        cal = rk.calibrate(K, dev(w["Qw"]), cfg.rank, fl, want_full=True)
    torch.cuda.synchronize()
    print(name, "ok", cal["info"].cpu().tolist()[:4])
