"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2605_19218_b200 as rk
from workload import CONFIGS, make_workload
from workload.gen import draw_v0

def dev(t):
    return torch.from_numpy(np.ascontiguousarray(t.bits).view(np.int16)).view(torch.bfloat16).cuda()

for cfg in (CONFIGS["llava_b1"].with_(h_kv=2, n_vis=300, n_text=20),
            CONFIGS["qwen_b1_r32"].with_(h_kv=1, n_vis=200, n_text=40),
            CONFIGS["toy"].with_(n_text=5)):
    w = make_workload(cfg)
    K = dev(w["K"])
    cal = rk.calibrate(K, dev(w["Qw"]), cfg.rank)
    sub = rk.calibrate_subspace(K, dev(w["Qw"]), torch.from_numpy(draw_v0(cfg)).cuda())
    Kc = rk.compress_kv(K, cal["R"])
    for kern in (0, 1):
        out = rk.decode_attn(dev(w["q"]), Kc, dev(w["V"]), cal["R"], cal["dmu"], dev(w["Ktext"]),
                             dev(w["Vtext"]), kernel=kern)
    torch.cuda.synchronize()
    print(cfg.name, "ok", float(out.abs().max()))
