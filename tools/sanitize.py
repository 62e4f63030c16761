"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck), plus the
GQA ring kernel on shapes that hit each of its CTA-count plans and merge paths, and the
token-selection prefill (r2)."""
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
    args = (dev(w["q"]), Kc, dev(w["V"]), cal["R"], cal["dmu"], dev(w["Ktext"]), dev(w["Vtext"]))
    for kern in (0, 1, 3, 4, 5):
        if kern in (3, 5) and (cfg.group < 2 or cfg.head_dim != 128):
            continue
        if kern == 4 and cfg.head_dim != 128:
            continue
        out = rk.decode_attn(*args, kernel=kern)
        # variable per-unit lengths (masked tiles, all-padding tiles skipped)
        nv = torch.tensor([max(1, cfg.n_vis - 37 * u) for u in range(cfg.units)], dtype=torch.int32).cuda()
        nt = torch.tensor([(cfg.n_text * u) // max(1, cfg.units) for u in range(cfg.units)],
                          dtype=torch.int32).cuda()
        rk.decode_attn(*args, kernel=kern, n_vis_u=nv, n_text_u=nt)
    # token shards (partial states + merge), offline state + shared rotation
    half = cfg.n_vis // 2
    parts = torch.stack([rk.decode_attn_partial(args[0], Kc[:, :half].contiguous(), args[2][:, :half].contiguous(),
                                                cal["R"], cal["dmu"]),
                         rk.decode_attn_partial(args[0], Kc[:, half:].contiguous(), args[2][:, half:].contiguous(),
                                                cal["R"], cal["dmu"], args[5], args[6])])
    rk.merge_partials(parts)
    st = rk.calib_accumulate(K, dev(w["Qw"]), rk.calib_state(cfg.h_kv, cfg.head_dim))
    off = rk.calibrate_from_state(st, cfg.rank)
    rk.compress_kv(K, off["R"])
    torch.cuda.synchronize()
    print(cfg.name, "ok", float(out.abs().max()))

# GQA ring plans: equal unit pieces with last-arriver / first-CTA merges (U = 8, 32), whole units
# per CTA (U = 160 -> 80 CTAs x 2), ranges inside units (U = 150); r = 64 (two R-chunks)
for U, N, M, r in ((8, 1500, 40, 32), (32, 700, 16, 32), (160, 200, 8, 32), (150, 300, 0, 32), (12, 900, 30, 64)):
    G, d = 7, 128
    g = torch.Generator(device="cuda").manual_seed(U + N)
    a = (torch.randn(U, G, d, device="cuda", generator=g).bfloat16(),
         torch.randn(U, N, r, device="cuda", generator=g).bfloat16(),
         torch.randn(U, N, d, device="cuda", generator=g).bfloat16(),
         torch.randn(U, d, r, device="cuda", generator=g) * 0.1, torch.randn(U, d, device="cuda", generator=g) * 0.1,
         torch.randn(U, M, d, device="cuda", generator=g).bfloat16() if M else None,
         torch.randn(U, M, d, device="cuda", generator=g).bfloat16() if M else None)
    o3 = rk.decode_attn(*a, kernel=3)
    rk.decode_attn_partial(*a)
    nv = torch.tensor([max(1, N - 97 * u) for u in range(U)], dtype=torch.int32).cuda()
    rk.decode_attn(*a, kernel=3, n_vis_u=nv)
    torch.cuda.synchronize()
    print("ring", U, N, M, r, "ok", float(o3.abs().max()))
# token-selection prefill (keep list and per-unit counts)
cfg = CONFIGS["llava_b1"].with_(h_kv=2, n_vis=400, n_text=0)
w = make_workload(cfg)
K = dev(w["K"])
keep = torch.sort(torch.randperm(cfg.n_vis)[:150]).values.to(torch.int32)
tok = torch.stack([keep] * cfg.units).cuda()
ct = rk.calibrate(K, dev(w["Qw"]), cfg.rank, tok_idx=tok)
rk.compress_kv(K, ct["R"], tok_idx=tok)
nvu = torch.tensor([400 - 111 * u for u in range(cfg.units)], dtype=torch.int32).cuda()
cu = rk.calibrate(K, dev(w["Qw"]), cfg.rank, n_vis_u=nvu)
rk.compress_kv(K, cu["R"], n_vis_u=nvu)
torch.cuda.synchronize()
print("tokens ok")
