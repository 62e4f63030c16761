#!/usr/bin/env python
"""Gap between consecutive ring-decode launches on one stream: launch 1 traced into buffer A,
launch 2 into buffer B; gap = first CTA start of launch 2 - last flusher/consumer end of 1."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19218_b200 as rk  # noqa: E402

U, G, N, M, r = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,7,4096,128,32").split(","))
kernel = int(sys.argv[2]) if len(sys.argv) > 2 else 3
d = 128
lay = []
for _ in range(3):
    lay.append((torch.randn(U, G, d, device="cuda").bfloat16(), torch.randn(U, N, r, device="cuda").bfloat16(),
                torch.randn(U, N, d, device="cuda").bfloat16(), torch.randn(U, d, r, device="cuda") * 0.1,
                torch.randn(U, d, device="cuda") * 0.1, torch.randn(U, M, d, device="cuda").bfloat16(),
                torch.randn(U, M, d, device="cuda").bfloat16(), torch.empty(U, G, d, device="cuda")))
for l in lay:
    rk.decode_attn(*l[:7], out=l[7], kernel=kernel)
torch.cuda.synchronize()
bufs = [torch.zeros(148 * 16, dtype=torch.int64, device="cuda") for _ in lay]
for _ in range(3):
    for l, b in zip(lay, bufs):
        b.zero_()
    torch.cuda.synchronize()
    for l, b in zip(lay, bufs):
        rk.debug_decode_trace(b)
        rk.decode_attn(*l[:7], out=l[7], kernel=kernel)
    rk.debug_decode_trace(None)
    torch.cuda.synchronize()
    ts = [b.view(148, 16).cpu() for b in bufs]
    starts = [t[t[:, 0] > 0, 0].min().item() for t in ts]
    ends = [max(t[t[:, 3] > 0, 3].max().item(), t[t[:, 4] > 0, 4].max().item() if (t[:, 4] > 0).any() else 0) for t in ts]
    print("launch spans (us):", [round((e - s) / 1e3, 2) for s, e in zip(starts, ends)],
          " gaps (us):", [round((starts[i + 1] - ends[i]) / 1e3, 2) for i in range(len(ts) - 1)])
