import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import numpy as np, torch
import paper_2605_19218_b200 as rk
from helpers import to_np64, to_torch
from workload import CONFIGS, make_workload
cfg = CONFIGS["llava_b1"].with_(h_kv=3, n_vis=300, n_text=0)
w = make_workload(cfg, dist="gap")
K = to_torch(w["K"]).clone()
K[1, :, 7] = 1.25; K[2, :, 3] = 0.0; K[2, :, 90] = 0.0
for name, fl in [("one", rk.DEFAULT_FLAGS), ("two", rk.DEFAULT_FLAGS | rk.EIG_TWOSIDED)]:
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, fl, want_full=True)
    torch.cuda.synchronize()
    Rf = to_np64(cal["R_full"]); lam = to_np64(cal["eigvals"])
    for u in range(3):
        M = Rf[u].T @ Rf[u] - np.eye(128)
        i, j = np.unravel_index(np.abs(M).argmax(), M.shape)
        print(name, u, "info", cal["info"][u].item(), "orth %.2e" % np.linalg.norm(M), "worst", i, j, "%.2e" % M[i, j],
              "lam_i %.3e lam_j %.3e" % (lam[u][i], lam[u][j]), "nzero lam", int((np.abs(lam[u]) < 1e-9 * np.abs(lam[u]).max()).sum()))
