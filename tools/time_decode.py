#!/usr/bin/env python
"""Decode timing sweeps (experiments; not the bench contract).

    python tools/time_decode.py "U,G,N,M,r" ...   (default: the GQA sweep below)

Random bf16 caches made on the device (timing only, no parity), L distinct layers per
graph replay so nothing is L2-resident; prints us/launch and GB/s of algorithmic bytes.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_19218_b200 as rk  # noqa: E402


def alg_bytes(U, G, N, M, r, d=128, s=2):
    return U * N * r * s + U * N * d * s + 2 * U * M * d * s + U * d * r * 4 + U * d * 4 + \
        U * G * d * s + U * G * d * 4


def time_shape(U, G, N, M, r, d=128, reps=30, kernel=0):
    kernel |= int(os.environ.get("TD_OVERLAP", "0")) * rk.DECODE_OVERLAP
    b = alg_bytes(U, G, N, M, r)
    L = max(2, min(16, int(600e6 // b) + 1))
    dev = "cuda"
    layers = []
    for _ in range(L):
        q = torch.randn(U, G, d, device=dev).bfloat16()
        Kc = torch.randn(U, N, r, device=dev).bfloat16()
        V = torch.randn(U, N, d, device=dev).bfloat16()
        R = torch.randn(U, d, r, device=dev) * 0.1
        dmu = torch.randn(U, d, device=dev) * 0.1
        Kt = torch.randn(U, M, d, device=dev).bfloat16() if M else None
        Vt = torch.randn(U, M, d, device=dev).bfloat16() if M else None
        out = torch.empty(U, G, d, device=dev)
        layers.append((q, Kc, V, R, dmu, Kt, Vt, out))
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # the layers were drawn on the default stream
    with torch.cuda.stream(s):
        ws = rk.workspace(rk.make_dims(U, G, d, r, N, M), rk.OP_DECODE, dev)
        for lay in layers:  # warm (attributes, descriptors)
            rk.decode_attn(*lay[:7], out=lay[7], ws=ws, kernel=kernel, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for lay in layers:
                rk.decode_attn(*lay[:7], out=lay[7], ws=ws, kernel=kernel, stream=s)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / L)
    ts.sort()
    us = ts[len(ts) // 2]
    return us, b / us / 1e3


def trace_shape(U, G, N, M, r, d=128, kernel=0):
    """One decode launch (after a warm launch on another layer) with per-warp stamps."""
    dev = "cuda"
    lay = []
    for _ in range(2):
        lay.append((torch.randn(U, G, d, device=dev).bfloat16(),
                    torch.randn(U, N, r, device=dev).bfloat16(),
                    torch.randn(U, N, d, device=dev).bfloat16(),
                    torch.randn(U, d, r, device=dev) * 0.1, torch.randn(U, d, device=dev) * 0.1,
                    torch.randn(U, M, d, device=dev).bfloat16() if M else None,
                    torch.randn(U, M, d, device=dev).bfloat16() if M else None,
                    torch.empty(U, G, d, device=dev)))
    ws = rk.workspace(rk.make_dims(U, G, d, r, N, M), rk.OP_DECODE, dev)
    buf = torch.zeros(148 * 16 * 8, dtype=torch.int64, device=dev)
    for lay_ in lay:
        rk.decode_attn(*lay_[:7], out=lay_[7], ws=ws, kernel=kernel)
    torch.cuda.synchronize()
    rk.debug_decode_trace(buf)
    rk.decode_attn(*lay[0][:7], out=lay[0][7], ws=ws, kernel=kernel)
    rk.decode_attn(*lay[1][:7], out=lay[1][7], ws=ws, kernel=kernel)
    torch.cuda.synchronize()
    rk.debug_decode_trace(None)
    t = buf.view(-1, 8).cpu()
    t = t[t[:, 0] > 0]
    t0 = int(t[:, 0].min())
    rel = (t[:, :5] - t0).double() / 1e3
    q = torch.tensor([0.0, 0.5, 0.9, 1.0], dtype=torch.double)
    names = ["start", "rotated", "tile0", "loopend", "end"]
    print(f"trace U={U} G={G} N={N} M={M} r={r} kernel={kernel}: warps={t.shape[0]} "
          f"tiles/warp {t[:, 5].double().mean():.1f} units/CTA max {int(t[:, 6].max())}")
    for k, nm in enumerate(names):
        v = torch.quantile(rel[:, k], q).tolist()
        print(f"   {nm:8s} min {v[0]:7.2f}  med {v[1]:7.2f}  p90 {v[2]:7.2f}  max {v[3]:7.2f} us")
    # stream time (tile0 -> loopend) by number of units touched, and by SM (warps / SM)
    st = rel[:, 3] - rel[:, 2]
    for nu in sorted(set(t[:, 6].tolist())):
        sel = t[:, 6] == nu
        print(f"   units={nu}: n={int(sel.sum())} stream med {st[sel].median():.2f} max {st[sel].max():.2f}"
              f"  loopend med {rel[sel, 3].median():.2f}")
    wps = t.shape[0] // 148 if t.shape[0] % 148 == 0 else 0
    if wps:
        per_sm = rel[:, 3].view(148, wps)
        smmax = per_sm.max(1).values
        smmin = per_sm.min(1).values
        print(f"   per-SM loopend: max-over-warps spread {smmax.min():.2f}..{smmax.max():.2f}; "
              f"within-SM spread med {(smmax - smmin).median():.2f} max {(smmax - smmin).max():.2f}")
        order = torch.argsort(smmax)
        print("   slowest SMs:", order[-8:].tolist(), " fastest:", order[:8].tolist())


def trace_ring(U, G, N, M, r, d=128):
    """The CTA-ring GQA kernel (kernel 3): 16 stamps per CTA (decode_ring.cuh) -> phase
    times of the first unit boundary inside a CTA's range."""
    dev = "cuda"
    lay = []
    for _ in range(2):
        lay.append((torch.randn(U, G, d, device=dev).bfloat16(),
                    torch.randn(U, N, r, device=dev).bfloat16(),
                    torch.randn(U, N, d, device=dev).bfloat16(),
                    torch.randn(U, d, r, device=dev) * 0.1, torch.randn(U, d, device=dev) * 0.1,
                    torch.randn(U, M, d, device=dev).bfloat16() if M else None,
                    torch.randn(U, M, d, device=dev).bfloat16() if M else None,
                    torch.empty(U, G, d, device=dev)))
    ws = rk.workspace(rk.make_dims(U, G, d, r, N, M), rk.OP_DECODE, dev)
    buf = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
    for lay_ in lay:
        rk.decode_attn(*lay_[:7], out=lay_[7], ws=ws, kernel=3)
    torch.cuda.synchronize()
    rk.debug_decode_trace(buf)
    rk.decode_attn(*lay[0][:7], out=lay[0][7], ws=ws, kernel=3)
    rk.decode_attn(*lay[1][:7], out=lay[1][7], ws=ws, kernel=3)
    torch.cuda.synchronize()
    rk.debug_decode_trace(None)
    t = buf.view(-1, 16).cpu()
    if os.environ.get("TD_DUMP"):
        torch.save(t, os.environ["TD_DUMP"])
    t = t[t[:, 0] > 0].double()
    t0 = t[:, 0].min()
    rel = lambda k: (t[:, k] - t0) / 1e3  # noqa: E731
    q = torch.tensor([0.0, 0.5, 0.9, 1.0], dtype=torch.double)
    tpu = -(-N // 64) + -(-M // 32)
    T = U * tpu
    C = t.shape[0]
    print(f"ring trace U={U} G={G} N={N} M={M} r={r}: CTAs={C} tiles/CTA {T / C:.1f}")
    for k, nm in [(13, "R0 landed"), (14, "R last landed"), (9, "rot0 partial"), (15, "rot0 bar"), (1, "rotated"), (2, "tile0"), (8, "u0 g0 done"),
                  (12, "u0 g1 done"), (10, "u0 ticket"), (11, "u1 tile0"), (3, "consumers end"),
                  (4, "flusher end")]:
        v = rel(k)
        v = v[t[:, k] > 0]
        if v.numel() == 0:
            continue
        qq = torch.quantile(v, q).tolist()
        print(f"   {nm:11s} min {qq[0]:7.2f}  med {qq[1]:7.2f}  p90 {qq[2]:7.2f}  max {qq[3]:7.2f} us  (n={v.numel()})")
    two = t[:, 6] >= 2
    if two.any():
        c = torch.arange(C, dtype=torch.double)[two]
        kA = torch.floor(c * T / C)
        kB = torch.floor((c + 1) * T / C)
        u0_tiles = torch.minimum(kB, (torch.floor(kA / tpu) + 1) * tpu) - kA
        u1_tiles = (kB - kA) - u0_tiles
        r0 = u0_tiles / (rel(8)[two] - rel(2)[two])
        r1 = u1_tiles / (rel(3)[two] - rel(11)[two])
        print(f"   2-unit CTAs: unit-0 tiles med {u0_tiles.median():.0f}; tiles/us unit 0 med {r0.median():.2f}, "
              f"unit 1 med {r1.median():.2f};  boundary (g0 done -> u1 tile0) med "
              f"{(rel(11)[two] - rel(8)[two]).median():.2f} us; flush med {(rel(9)[two] - rel(8)[two]).median():.2f}; "
              f"g1 - g0 done med {(rel(12)[two] - rel(8)[two]).median():.2f}")
    one = t[:, 6] == 1
    if one.any():
        c = torch.arange(C, dtype=torch.double)[one]
        n = torch.floor((c + 1) * T / C) - torch.floor(c * T / C)
        print(f"   1-unit CTAs: tiles/us med {(n / (rel(3)[one] - rel(2)[one])).median():.2f}")


def trace_repeat(U, G, N, M, r, d=128, reps=3):
    """Is the per-warp finish time systematic?  Same launch traced `reps` times."""
    dev = "cuda"
    lay = (torch.randn(U, G, d, device=dev).bfloat16(), torch.randn(U, N, r, device=dev).bfloat16(),
           torch.randn(U, N, d, device=dev).bfloat16(), torch.randn(U, d, r, device=dev) * 0.1,
           torch.randn(U, d, device=dev) * 0.1,
           torch.randn(U, M, d, device=dev).bfloat16() if M else None,
           torch.randn(U, M, d, device=dev).bfloat16() if M else None, torch.empty(U, G, d, device=dev))
    ws = rk.workspace(rk.make_dims(U, G, d, r, N, M), rk.OP_DECODE, dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    ends, sms = [], []
    for i in range(reps + 1):
        os.environ["ROTATEK_CTA_ROT"] = str(0 if i < 2 else 37 * (i - 1))
        buf = torch.zeros(148 * 16 * 8, dtype=torch.int64, device=dev)
        flush.fill_(i)
        torch.cuda.synchronize()
        rk.debug_decode_trace(buf)
        rk.decode_attn(*lay[:7], out=lay[7], ws=ws)
        torch.cuda.synchronize()
        rk.debug_decode_trace(None)
        t = buf.view(-1, 8).cpu()
        t = t[t[:, 0] > 0]
        ends.append(((t[:, 3] - t[:, 0].min()) - (t[:, 2] - t[:, 0].min())).double() / 1e3)
        sms.append(t[:, 7].clone())
    e = torch.stack(ends[1:])
    c = torch.corrcoef(e)
    print(f"repeat U={U} G={G} N={N}: stream-time corr between launches:\n{c}")
    print(f"   per-warp mean over launches: spread {e.mean(0).min():.2f}..{e.mean(0).max():.2f}, "
          f"per-launch spreads {[round(float(x.max() - x.min()), 2) for x in e]}")
    # by warp index within SM (w % 8) and by SM
    wm = e.mean(0)
    print("   by warp-in-CTA:", [round(float(wm[k::8].mean()), 2) for k in range(8)])
    same = [float((sms[i] == sms[i + 1]).double().mean()) for i in range(1, reps)]
    print(f"   fraction of warps on the same SM as in the previous launch: {same}")
    # per-SM mean stream time in each launch: is slowness attached to the SM?
    per = []
    for i in range(1, reps + 1):
        v = torch.zeros(160, dtype=torch.double)
        n = torch.zeros(160, dtype=torch.double)
        v.index_add_(0, sms[i].long(), e[i - 1])
        n.index_add_(0, sms[i].long(), torch.ones_like(e[i - 1]))
        per.append(v[:148] / n[:148].clamp(min=1))
    print(f"   per-SM mean stream time corr between launches: {torch.corrcoef(torch.stack(per))[0, 1:].tolist()}")


def main():
    kern = int(os.environ.get("TD_KERNEL", "0"), 0)
    if kern:
        global time_shape
        base_fn = time_shape
        time_shape = lambda *a, **k: base_fn(*a, kernel=kern, **k)  # noqa: E731
    if sys.argv[1:2] == ["--repeat"]:
        for sh in sys.argv[2:]:
            trace_repeat(*(int(x) for x in sh.split(",")))
        return
    if sys.argv[1:2] == ["--trace-ring"]:
        for sh in sys.argv[2:]:
            trace_ring(*(int(x) for x in sh.split(",")))
        return
    if sys.argv[1:2] == ["--trace"]:
        for sh in sys.argv[2:]:
            trace_shape(*(int(x) for x in sh.split(",")[:5]),
                        kernel=int(sh.split(",")[5]) if sh.count(",") >= 5 else 0)
        return
    shapes = sys.argv[1:] or [
        "128,7,4096,128,32", "128,7,1024,128,32", "128,7,2048,128,32", "128,7,8192,128,32",
        "128,7,16384,128,32", "128,7,4096,0,32", "32,7,4096,128,32", "512,7,4096,128,32",
        "64,7,32768,128,32", "128,7,4096,128,64", "128,1,4096,128,32", "2048,1,864,128,32",
        "1024,1,2880,128,32", "128,7,64,0,32", "1024,1,64,0,32"]
    for sh in shapes:
        U, G, N, M, r = (int(x) for x in sh.split(","))
        us, gbs = time_shape(U, G, N, M, r)
        print(f"U={U:5d} G={G} N={N:6d} M={M:4d} r={r:3d}  {us:9.2f} us  {gbs:8.1f} GB/s  "
              f"bytes={alg_bytes(U, G, N, M, r) / 1e6:.1f} MB", flush=True)


if __name__ == "__main__":
    main()
