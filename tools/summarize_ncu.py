#!/usr/bin/env python
"""Summarise ncu captures from tools/profile_all.sh (markdown tables on stdout).

    python tools/summarize_ncu.py --tag r2a [--src gpurun_out] [--write-traffic]

--write-traffic MERGES the decode captures found for the tag into profiles/ncu_traffic.json
(dram bytes per decode launch, read by bench.py for roofline.traffic); configs without a
capture keep their entries.  Without it nothing is written."""
import argparse
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workload import CONFIGS, decode_bytes  # noqa: E402

ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
ap.add_argument("--tag", required=True, help="capture tag, e.g. r2a (file names *_<tag>_raw.csv)")
ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
ap.add_argument("--write-traffic", action="store_true", help="merge into profiles/ncu_traffic.json")
opt = ap.parse_args()
tag, src = opt.tag, opt.src

WANT = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__bytes_read.sum.pct_of_peak_sustained_elapsed": "dram_read_pct",
    "dram__bytes_write.sum.pct_of_peak_sustained_elapsed": "dram_write_pct",
    "dram__bytes.sum.per_second": "dram_bps",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed": "utc_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "sm_issue_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_hmma_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_pct",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active": "uniform_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def raw_rows(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    out = []
    for r in rows[2:]:  # row 1 holds units
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")}
        units = dict(zip(hdr, rows[1]))
        for k, v in WANT.items():
            if k in d and d[k] not in ("", "n/a"):
                try:
                    x = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                u = units.get(k, "")
                if k == "gpu__time_duration.sum" and u == "ms":
                    x *= 1e6
                elif k == "gpu__time_duration.sum" and u == "us":
                    x *= 1e3
                if k == "dram__bytes.sum.per_second":
                    x *= {"Tbyte/s": 1e12, "Gbyte/s": 1e9, "Mbyte/s": 1e6}.get(u, 1.0)
                if k.startswith("dram__bytes") and u == "Mbyte":
                    x *= 1e6
                elif k.startswith("dram__bytes") and u == "Gbyte":
                    x *= 1e9
                elif k.startswith("dram__bytes") and u == "Kbyte":
                    x *= 1e3
                rec[v] = x
        rec["dram_pct"] = rec.get("dram_read_pct", 0.0) + rec.get("dram_write_pct", 0.0)
        out.append(rec)
    return out


tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
traffic["_source"] = ("ncu --set full --clock-control none (tools/profile_all.sh), one decode launch, "
                      "dram__bytes_read.sum + dram__bytes_write.sum; per-config 'capture' names the file")
lines = ["| config | kernel | ncu time (us) | dram read+write (MB) | alg. bytes (MB) | traffic/alg | "
         "DRAM % peak | SM issue % | regs |", "|---|---|---|---|---|---|---|---|---|"]
for cfg in ("llava_b32", "qwen_b32_r32", "joint_b64", "long_b16", "qwen_b32_r64", "llava_b8", "qwen_b8_r32"):
    p = os.path.join(src, f"ncu_decode_{cfg}_{tag}_raw.csv")
    if not os.path.exists(p):
        continue
    recs = raw_rows(p)
    if not recs:
        continue
    r = recs[0]
    alg = decode_bytes(CONFIGS[cfg])
    tot = r.get("dram_read", 0) + r.get("dram_write", 0)
    traffic[cfg] = {"dram_bytes_per_launch": int(tot), "dram_read": int(r.get("dram_read", 0)),
                    "dram_write": int(r.get("dram_write", 0)), "algorithmic_bytes_per_launch": alg,
                    "kernel": r["kernel"][:80], "capture": f"profiles/ncu_decode_{cfg}_{tag}_details.csv"}
    lines.append(f"| {cfg} | {r['kernel'][:40]} | {r.get('time', 0) / 1e3:.1f} | {tot / 1e6:.1f} | "
                 f"{alg / 1e6:.1f} | {tot / alg:.3f} | {r.get('dram_pct', 0):.1f} | "
                 f"{r.get('sm_issue_pct', r.get('issue_pct', 0)):.1f} | {int(r.get('regs', 0))} |")
if opt.write_traffic:
    json.dump(traffic, open(tpath, "w"), indent=1)
print("\n".join(lines))

p = os.path.join(src, f"ncu_prefill_llava_b32_{tag}_raw.csv")
if os.path.exists(p):
    print("\n| prefill kernel (llava_b32) | ncu time (us) | dram MB | DRAM % | L1/smem % | SM issue % | tensor pipe % | regs | grid x block |")
    print("|---|---|---|---|---|---|---|---|---|")
    seen = set()
    for r in raw_rows(p):
        k = r["kernel"].split("(")[0]
        if k in seen:
            continue
        seen.add(k)
        tc = r.get("tensor_pct", r.get("utc_pct", 0))
        print(f"| {k[:48]} | {r.get('time', 0) / 1e3:.1f} | {(r.get('dram_read', 0) + r.get('dram_write', 0)) / 1e6:.1f} | "
              f"{r.get('dram_pct', 0):.1f} | {r.get('l1_pct', 0):.1f} | {r.get('sm_issue_pct', 0):.1f} | {tc:.1f} | "
              f"{int(r.get('regs', 0))} | {int(r.get('grid', 0))}x{int(r.get('block', 0))} |")

# launch lists: share of the decode kernel in one bench step
print("\n| config | launches | decode share of step (ncu, serialised) | top kernels (us) |")
print("|---|---|---|---|")
for cfg in ("llava_b32", "qwen_b32_r32", "joint_b64", "long_b16", "qwen_b32_r64", "llava_b8", "qwen_b8_r32"):
    p = os.path.join(src, f"launches_{cfg}_{tag}.csv")
    if not os.path.exists(p):
        continue
    t = defaultdict(float)
    n = 0
    for r in csv.reader(open(p)):
        if len(r) > 14 and r[0].isdigit() and "rk::" in r[4]:
            k = r[4].split("(")[0].replace("void ", "").replace("rk::", "")
            k = k.split("<")[0]
            t[k] += float(r[14].replace(",", "")) / 1e3
            n += 1
    tot = sum(t.values())
    dec = sum(v for k, v in t.items() if k.startswith("decode"))
    top = ", ".join(f"{k} {v:.0f}" for k, v in sorted(t.items(), key=lambda x: -x[1])[:4])
    print(f"| {cfg} | {n} | {dec / tot:.4f} | {top} |")
