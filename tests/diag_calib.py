"""Diagnostics (test infrastructure, not a test): per-stage GPU vs oracle errors for a
config (prints, no asserts).  Lives under tests/ because only tests may use oracle/."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))  # tests/
import numpy as np, torch
import paper_2605_19218_b200 as rk
from oracle import oracle as orc
from workload import CONFIGS, make_workload
from helpers import to_torch, to_np64, max_rel_err

def run(cfg, dist="nat", units=None, **kw):
    w = make_workload(cfg, dist=dist, **kw)
    K = to_torch(w["K"])
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, want_full=True)
    Kc = rk.compress_kv(K, cal["R"])
    M = cfg.n_text
    out = rk.decode_attn(to_torch(w["q"]), Kc, to_torch(w["V"]), cal["R"], cal["dmu"],
                         to_torch(w["Ktext"]) if M else None, to_torch(w["Vtext"]) if M else None)
    torch.cuda.synchronize()
    ref = orc.pipeline(w["K"].f64(), w["V"].f64(), w["Qw"].f64(), w["q"].f64(), cfg.rank, cfg.dtype,
                       w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None)
    R = to_np64(cal["R"]); lam = to_np64(cal["eigvals"])
    print(f"== {cfg.name} dist={dist} {kw} dtype={cfg.dtype} info={cal['info'].tolist()[:8]}")
    for u in range(min(cfg.units, 4)):
        P = R[u] @ R[u].T; Pr = ref["R"][u] @ ref["R"][u].T
        Cq = ref["Cq"][u]; nrm = np.linalg.norm(Cq)
        D = R[u].T @ Cq @ R[u]
        ls = np.sort(ref["lam"][u])[::-1]
        gl = np.sort(lam[u])[::-1]
        print(f" u{u}: |P-Pref|={np.linalg.norm(P-Pr):.2e} orth={np.linalg.norm(R[u].T@R[u]-np.eye(cfg.rank)):.2e}"
              f" offdiag={np.linalg.norm(D-np.diag(np.diag(D)))/nrm:.2e} trace_rel={abs(lam[u].sum()-np.trace(Cq))/abs(np.trace(Cq)):.2e}"
              f" cap={np.trace(D)/ls[:cfg.rank].sum():.8f} gap={ls[cfg.rank-1]/ls[cfg.rank]:.3f} lamerr={np.abs(gl-ls).max()/ls[0]:.2e}")
    Rref = ref["R"]
    dmu_ref = orc.dmu_from_R(R, ref["mu"])
    print(" dmu err", np.abs(to_np64(cal["dmu"]) - dmu_ref).max(), "dmu scale", np.abs(dmu_ref).max())
    want = orc.quantize(orc.compress(w["K"].f64(), R), cfg.dtype)
    got = to_np64(Kc)
    print(" compress exact frac", np.mean(got == want), "max rel", (np.abs(got-want)/np.maximum(np.abs(want),1e-30)).max())
    print(" e2e err", max_rel_err(to_np64(out), ref["out"]))
    dec = orc.decode(w["q"].f64(), got, w["V"].f64(), R, to_np64(cal["dmu"]),
                     w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None)
    print(" decode-on-gpu-bytes err", max_rel_err(to_np64(out), dec))
    # oracle with GPU's R (as stored) but its own K~
    dec2 = orc.decode(w["q"].f64(), orc.quantize(orc.compress(w["K"].f64(), R), cfg.dtype), w["V"].f64(), R,
                      orc.dmu_from_R(R, ref["mu"]), w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None)
    print(" as-stored oracle vs fp64 oracle", max_rel_err(dec2, ref["out"]))
    # sharpness
    s = orc.scores(w["q"].f64(), ref["Kt"], ref["R"], ref["dmu"], w["Ktext"].f64() if M else None)
    p = np.exp(s - s.max(-1, keepdims=True)); p /= p.sum(-1, keepdims=True)
    print(" N_eff (1/sum p^2) median", np.median(1/(p**2).sum(-1)), "min", (1/(p**2).sum(-1)).min())

for dt in ("bf16", "f32"):
    run(CONFIGS["llava_b1"].with_(h_kv=4, n_vis=777, n_text=0, dtype=dt), dist="gap", mean=0.5)
    run(CONFIGS["llava_b1"].with_(h_kv=4, n_vis=777, n_text=0, dtype=dt), dist="gap", mean=20.0)
run(CONFIGS["llava_b1"].with_(h_kv=4))
run(CONFIGS["qwen_b1_r32"])
run(CONFIGS["long_b16"].with_(batch=1))
