#!/usr/bin/env python
"""One calibrate (Jacobi) + one calibrate_subspace + one compress call on a config, for ncu
launch lists and captures.
    ncu --metrics gpu__time_duration.sum python tools/prof_calib.py llava_b32"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19218_b200 as rk  # noqa: E402
from workload import CONFIGS, make_workload  # noqa: E402
from workload.gen import draw_v0  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "llava_b32"]
w = make_workload(cfg, threads=os.cpu_count() or 8)


def dev(t):
    return torch.from_numpy(np.ascontiguousarray(t.bits).view(np.int16)).view(torch.bfloat16).cuda()


K, Qw = dev(w["K"]), dev(w["Qw"])
V0 = torch.from_numpy(draw_v0(cfg)).cuda()
cal = rk.calibrate(K, Qw, cfg.rank)
rk.calibrate_subspace(K, Qw, V0)
rk.compress_kv(K, cal["R"])
torch.cuda.synchronize()
print("done")
