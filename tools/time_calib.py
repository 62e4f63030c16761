"""Time rotatek_calibrate phases for a config with different flags (experiments)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_19218_b200 as rk
from workload import CONFIGS, make_workload

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llava_b32"]
w = make_workload(cfg, threads=os.cpu_count() or 8)
def dev(t):
    return torch.from_numpy(np.ascontiguousarray(t.bits).view(np.int16)).view(torch.bfloat16).cuda()
K, Qw = dev(w["K"]), dev(w["Qw"])
for name, flags in [("fp32-onesided-jacobi+fp64-refine", rk.DEFAULT_FLAGS),
                    ("fp32-twosided-jacobi+fp64-refine", rk.DEFAULT_FLAGS | rk.EIG_TWOSIDED),
                    ("fp64-jacobi", rk.DEFAULT_FLAGS | rk.EIG_FP64)]:
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        cal = rk.calibrate(K, Qw, cfg.rank, flags)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    info = cal["info"].cpu().numpy()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    Kc = rk.compress_kv(K, cal["R"])
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"   compress: {1e3*(t3-t2):.3f} ms (host-timed)")
    print(f"{cfg.name} {name}: {1e3*(t1-t0):.2f} ms  info>0: {(info>0).sum()}  info<0: {(info<0).sum()}")

from workload.gen import draw_v0
V0 = torch.from_numpy(draw_v0(cfg)).cuda()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cal = rk.calibrate_subspace(K, Qw, V0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"{cfg.name} subspace(T=5): {1e3*(t1-t0):.2f} ms  info<0: {(cal['info'].cpu().numpy()<0).sum()}")

# one-sided vs two-sided Jacobi on every unit: top-r projector distance, eigenvalue agreement
a = rk.calibrate(K, Qw, cfg.rank, rk.DEFAULT_FLAGS, want_full=True)
b = rk.calibrate(K, Qw, cfg.rank, rk.DEFAULT_FLAGS | rk.EIG_TWOSIDED, want_full=True)
Ra, Rb = a["R"].double(), b["R"].double()
Pa, Pb = Ra @ Ra.transpose(1, 2), Rb @ Rb.transpose(1, 2)
dP = torch.linalg.matrix_norm(Pa - Pb).max().item()
la, lb = a["eigvals"].double().sort(-1).values, b["eigvals"].double().sort(-1).values
dl = ((la - lb).abs().max(-1).values / lb.abs().max(-1).values).max().item()
same_idx = bool((a["idx"] == b["idx"]).all().item())
print(f"one-sided vs two-sided: max |P_a - P_b|_F {dP:.3e}  max rel eig diff {dl:.3e}  idx equal {same_idx}  "
      f"info one-sided min/max {a['info'].min().item()}/{a['info'].max().item()}")
if os.environ.get("ROTATEK_HJ_SWEEPS"):
    inf = a["info"].cpu().numpy()
    print("one-sided sweeps (info - 1000): min", inf.min() - 1000, "max", inf.max() - 1000,
          "mean", round(float(inf.mean()) - 1000, 2))
