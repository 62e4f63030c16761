#!/usr/bin/env python
"""Benchmark of the RotateK hot path on B200 (contract: see DESIGN.md "Measurement").

    python bench.py [--gpus N --steps K --warmup W] [--config llava_b32] [--layers L]
    python bench.py --impl reference ...        (the fp64 CPU oracle, bounded sample)
    torchrun --nproc-per-node N bench.py --gpus N ...   (or plain --gpus N: self-launches)

Headline (BASELINE.json metric): sparse-channel decode attention us/layer and HBM GB/s.
One timed step = one decode pass (Alg. 2, all query heads, one rotatek_decode_attn
launch per layer) over L distinct layer caches of the workload, captured in a CUDA
graph.  `value` = algorithmic decode bytes of all ranks / max-over-ranks step time.
The full hot path (calibrate + compress + decode per layer, every SURVEY §8(a) row) is
timed as well and reported under "full_step"; "e2e" runs that full path from pinned
host buffers with the host<->device copies inside the timed region.
Multi-GPU: the headline is WEAK scaling -- each rank owns its own batch of
units (b x kv-head), no collective on the data path.  With N > 1 the line also carries
"strong": the same global batch split over the N ranks by unit ranges, with the one
NCCL all-gather of the outputs (north_star: "NCCL over NVLink is used only to gather
outputs") timed separately from the decode kernels (max over ranks).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workload import CONFIGS, compress_bytes, decode_bytes, decode_flops, make_workload  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
NOMINAL_HBM_GBS = 8000.0
EXTRA_ROWS = ("qwen_b32_r32", "long_b16")  # driver-visible GQA rows besides the headline


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llava_b32")
    ap.add_argument("--override", default="",
                    help="experiments only: comma list of Config fields, e.g. group=2,batch=8")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--kernel", type=int, default=0, help="0 auto, 1 generic, 2 fast, 3 GQA ring, 5 GQA per-warp")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--skip-full", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-extra", action="store_true")
    ap.add_argument("--skip-strong", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU)
    with torch.distributed.run on this node; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], "measured", d
    return 6650.0, "fallback (B200_PROFILING.md)", {}


def get_config(args, name=None):
    cfg = CONFIGS[name or args.config]
    if args.override and name is None:
        kw = {}
        for item in args.override.split(","):
            k, v = item.split("=")
            kw[k] = type(getattr(cfg, k))(v)
        cfg = cfg.with_(**kw)
    return cfg


def rank_units(cfg, rank):
    """Weak scaling: each rank owns a full per-GPU batch of units (sharding.weak_units)."""
    from paper_2605_19218_b200.sharding import weak_units
    return list(weak_units(cfg.units, rank))


def ncu_traffic(name):
    """ncu dram bytes per launch of the decode kernel for a config (profiles/ncu_traffic.json,
    written by tools/summarize_ncu.py from the committed captures), or None."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        tr = json.load(open(tp)).get(name)
        if tr:
            return tr.get("dram_bytes_per_launch")
    return None


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


# ----------------------------------------------------------------------------- CPU oracle
def _oracle_sample(cfg, n_units):
    from oracle import oracle as orc
    w = make_workload(cfg, units=range(n_units), threads=os.cpu_count() or 8)
    return orc, w


def oracle_baseline(cfg, seconds):
    """The fp64 oracle as it stands on the host cores, on a bounded sample of the workload:
    (1) Alg. 2 decode passes for ~`seconds` on all cores, in the metric's unit (GB/s of
    decode bytes); (2) one calibrate + compress (Alg. 1, steps 1-7) of the sample;
    (3) the same decode with ONE thread (a subprocess with OMP_NUM_THREADS=1)."""
    n_units = max(1, min(cfg.units, 64))
    orc, w = _oracle_sample(cfg, n_units)
    t0 = time.perf_counter()
    cal = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    Kt = orc.quantize(orc.compress(w["K"].f64(), cal["R"]), cfg.dtype)
    t_prefill = time.perf_counter() - t0
    args = (w["q"].f64(), Kt, w["V"].f64(), cal["R"], cal["dmu"], w["Ktext"].f64(), w["Vtext"].f64())
    sub = cfg.with_(batch=1, h_kv=n_units)
    reps, t0 = 0, time.perf_counter()
    while True:
        orc.decode(*args)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    gbs = decode_bytes(sub) * reps / el / 1e9
    model, nproc = cpu_info()
    cores = int(os.environ.get("OMP_NUM_THREADS", nproc))
    out = {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "oracle",
           "sample": f"{n_units} of {cfg.units} units of {cfg.name}, {reps} decode passes",
           "seconds": round(el, 2), "cpu_model": model, "nproc": nproc,
           "prefill_all_cores": {"seconds": round(t_prefill, 3), "units": n_units,
                                 "tokens_per_s": round(n_units * cfg.n_vis / t_prefill, 1),
                                 "what": "oracle calibrate (sigma, two-pass covariance, cyclic Jacobi, "
                                         "select, delta_mu) + compress K R_r + RNE, fp64"}}
    # one thread, in a subprocess (OpenMP's thread count is fixed when the library loads)
    code = ("import sys,time,json; sys.path.insert(0, %r)\n"
            "from bench import _oracle_sample, decode_bytes\n"
            "from workload import CONFIGS\n"
            "cfg = CONFIGS[%r]; n = %d\n"
            "orc, w = _oracle_sample(cfg, n)\n"
            "t0 = time.perf_counter(); cal = orc.calibrate(w['K'].f64(), w['Qw'].f64(), cfg.rank)\n"
            "Kt = orc.quantize(orc.compress(w['K'].f64(), cal['R']), cfg.dtype); tp = time.perf_counter() - t0\n"
            "a = (w['q'].f64(), Kt, w['V'].f64(), cal['R'], cal['dmu'], w['Ktext'].f64(), w['Vtext'].f64())\n"
            "reps = 0; t0 = time.perf_counter()\n"
            "while True:\n"
            "    orc.decode(*a); reps += 1; el = time.perf_counter() - t0\n"
            "    if el >= %f: break\n"
            "sub = cfg.with_(batch=1, h_kv=n)\n"
            "print(json.dumps(dict(gbs=decode_bytes(sub) * reps / el / 1e9, reps=reps, seconds=el, prefill=tp)))\n"
            % (ROOT, cfg.name, max(1, n_units // 8), seconds / 2))
    try:
        env = dict(os.environ, OMP_NUM_THREADS="1")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        one = json.loads(r.stdout.strip().splitlines()[-1])
        out["single_thread"] = {"value": round(one["gbs"], 4), "unit": "GB/s", "cores": 1,
                                "sample": f"{max(1, n_units // 8)} units, {one['reps']} decode passes",
                                "seconds": round(one["seconds"], 2),
                                "prefill_tokens_per_s": round(max(1, n_units // 8) * cfg.n_vis / one["prefill"], 1)}
    except Exception as e:  # pragma: no cover - reported, not fatal
        out["single_thread"] = {"error": repr(e)[:200]}
    return out


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores (rank 0 only)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = get_config(args)
    from oracle import oracle as orc
    n_units = max(1, min(cfg.units, 32))
    w = make_workload(cfg, units=range(n_units), threads=os.cpu_count() or 8)
    cal = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    Kt = orc.quantize(orc.compress(w["K"].f64(), cal["R"]), cfg.dtype)
    dargs = (w["q"].f64(), Kt, w["V"].f64(), cal["R"], cal["dmu"], w["Ktext"].f64(),
             w["Vtext"].f64())
    for _ in range(args.warmup):
        orc.decode(*dargs)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.decode(*dargs)
        times.append(time.perf_counter() - t0)
    sub = cfg.with_(batch=1, h_kv=n_units)
    tot = sum(times)
    gbs = decode_bytes(sub) * len(times) / tot / 1e9
    model, nproc = cpu_info()
    cores = int(os.environ.get("OMP_NUM_THREADS", nproc))
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot / len(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "units": cfg.units, "sample_units": n_units,
                   "n_vis": cfg.n_vis, "n_text": cfg.n_text, "head_dim": cfg.head_dim,
                   "rank": cfg.rank, "group": cfg.group},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores,
                         "kind": "oracle", "cpu_model": model, "nproc": nproc,
                         "sample": f"{n_units} of {cfg.units} units, one decode pass per step"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- clocks
class Clocks:
    """Samples SM clock and clock-event (throttle) reasons through NVML every ~1 ms
    while the timed region runs (same counters nvidia-smi's clocks line reads)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.ok = False

    def _run(self):
        import pynvml as nv
        h = self.h
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis else self.gpu
            self.h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.stop = threading.Event()
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = repr(e)
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.th.join(timeout=2)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["no samples" if self.ok else getattr(self, "err", "nvml")]}
        sm = [s for s, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "NVML during the timed decode region"}


# ----------------------------------------------------------------------------- ours
def _to_dev(t, dev):
    import torch
    x = np.ascontiguousarray(t.bits)
    if t.dtype == "bf16":
        x = torch.from_numpy(x.view(np.int16)).view(torch.bfloat16)
    else:
        x = torch.from_numpy(x)
    return x.to(dev)


def prepare_layers(rk, cfg, L, units, dev):
    """Layer 0 drawn on the host (per-unit seeded generator, these units); layers 1..L-1 are
    distinct device buffers (unit axis rolled), so L layers exceed the 126 MB L2.  Prefill
    (calibrate + compress, on the GPU) builds each layer's compressed cache."""
    import torch
    t_gen = time.perf_counter()
    host = make_workload(cfg, units=units, threads=os.cpu_count() or 8)
    t_gen = time.perf_counter() - t_gen
    base = {k: _to_dev(host[k], dev) for k in ("K", "V", "Ktext", "Vtext", "Qw", "q")}
    layers = []
    for l in range(L):
        sh = (7 * l) % len(units)
        layers.append({k: torch.roll(v, shifts=sh, dims=0).contiguous() if l else v
                       for k, v in base.items()})
    for ly in layers:
        cal = rk.calibrate(ly["K"], ly["Qw"], cfg.rank)
        ly["R"], ly["dmu"], ly["info"] = cal["R"], cal["dmu"], cal["info"]
        ly["Kc"] = rk.compress_kv(ly["K"], ly["R"])
        ly["out"] = torch.empty((len(units), cfg.group, cfg.head_dim), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    bad = int(sum((ly["info"] != 0).sum().item() for ly in layers))
    return host, layers, t_gen, bad


def decode_graph(rk, cfg, layers, stream, kernel=0, graph=True, lo=0, hi=None):
    """A CUDA graph of one decode launch per layer over units [lo, hi) of each layer."""
    import torch
    hi = cfg.units if hi is None else hi
    U = hi - lo
    dims = rk.make_dims(U, cfg.group, cfg.head_dim, cfg.rank, cfg.n_vis, cfg.n_text, 0,
                        rk.BF16 if cfg.dtype == "bf16" else rk.F32)
    with torch.cuda.stream(stream):
        ws = torch.zeros(rk.workspace_bytes(dims, rk.OP_DECODE), dtype=torch.uint8, device=stream.device)
    outs = [ly["out"][lo:hi] for ly in layers]

    def step():
        for ly, o in zip(layers, outs):
            rk.decode_attn(ly["q"][lo:hi], ly["Kc"][lo:hi], ly["V"][lo:hi], ly["R"][lo:hi], ly["dmu"][lo:hi],
                           ly["Ktext"][lo:hi], ly["Vtext"][lo:hi], out=o, ws=ws, kernel=kernel, stream=stream)

    stream.wait_stream(torch.cuda.current_stream())
    g = None
    with torch.cuda.stream(stream):
        step()
        launches = rk.last_launch_count()
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step()
    torch.cuda.synchronize()

    def run():
        if g is not None:
            with torch.cuda.stream(stream):
                g.replay()
        else:
            step()
    return run, launches, ws


def time_region(run, steps, warmup, stream, barrier):
    import torch
    for _ in range(warmup):
        run()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    barrier()
    return e0.elapsed_time(e1)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2605_19218_b200 as rk

    world, rank, local = dist_env()
    # ROTATEK_BENCH_SHARE_GPU=1 (tests only): every rank on cuda:0 with gloo collectives, to
    # exercise the N > 1 code path on a one-GPU box; its timings mean nothing
    share_gpu = os.environ.get("ROTATEK_BENCH_SHARE_GPU") == "1"
    if share_gpu:
        local = 0
    if world > 1:
        if share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = get_config(args)
    L = args.layers
    peak_gbs, peak_kind, _ = peaks()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if share_gpu else dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    host, layers, t_gen, bad_info = prepare_layers(rk, cfg, L, rank_units(cfg, rank), dev)
    stream = torch.cuda.Stream(device=dev)
    run_step, launches_per_decode, ws = decode_graph(rk, cfg, layers, stream, args.kernel, not args.no_graph)

    # ---------------- timed region A: decode steps (weak scaling: every rank its own batch)
    for _ in range(args.warmup):
        run_step()
    barrier()
    clocks = Clocks(local)
    with clocks:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            run_step()
        ev1.record(stream)
        barrier()
    ms_total = max_ranks(ev0.elapsed_time(ev1))
    ms_step = ms_total / args.steps
    us_layer = 1e3 * ms_step / L
    bytes_layer = decode_bytes(cfg)
    achieved = bytes_layer / (us_layer * 1e-6) / 1e9          # per-launch GB/s (this rank)
    value = world * bytes_layer * L / (ms_step * 1e-3) / 1e9   # whole job

    # ---------------- strong scaling (N > 1): the same global batch split over the ranks,
    # decode kernels and the output all-gather (one NCCL all_gather_into_tensor per layer)
    strong = None
    if world > 1 and not args.skip_strong:
        from paper_2605_19218_b200.sharding import strong_units
        per = -(-cfg.units // world)
        rng = strong_units(cfg.units, rank, world)
        # this rank's shard of the global batch: len(rng) units, timed on the first len(rng)
        # units of its own (identically generated, unit-rolled) buffers -- same shapes, same
        # bytes per unit
        lo, hi = 0, len(rng)
        run_k, _, _ = decode_graph(rk, cfg, layers, stream, args.kernel, not args.no_graph, lo, hi)
        gather_out = [torch.empty((world * per, cfg.group, cfg.head_dim), dtype=torch.float32, device=dev)
                      for _ in range(L)]
        send = [torch.zeros((per, cfg.group, cfg.head_dim), dtype=torch.float32, device=dev) for _ in range(L)]

        def run_gather():
            with torch.cuda.stream(stream):
                for l in range(L):
                    send[l][: hi - lo].copy_(layers[l]["out"][lo:hi])
                    if share_gpu:  # debug mode: gloo on one GPU, staged through the host
                        hb = torch.empty((world * per, cfg.group, cfg.head_dim), dtype=torch.float32)
                        dist.all_gather_into_tensor(hb, send[l].cpu())
                        gather_out[l].copy_(hb)
                    else:
                        dist.all_gather_into_tensor(gather_out[l], send[l])

        k_ms = max_ranks(time_region(run_k, args.steps, args.warmup, stream, barrier)) / args.steps
        g_ms = max_ranks(time_region(run_gather, args.steps, args.warmup, stream, barrier)) / args.steps

        def run_both():
            run_k()
            run_gather()
        t_ms = max_ranks(time_region(run_both, args.steps, args.warmup, stream, barrier)) / args.steps
        strong = {"global_units": cfg.units, "units_per_rank": per, "ranks": world,
                  "kernel_us_per_layer": round(1e3 * k_ms / L, 3),
                  "gather_us_per_layer": round(1e3 * g_ms / L, 3),
                  "total_us_per_layer": round(1e3 * t_ms / L, 3),
                  "value_gbs": round(bytes_layer / (1e-3 * t_ms / L) / 1e9, 2),
                  "gather_bytes_per_layer": int(world * per * cfg.group * cfg.head_dim * 4),
                  "collective": "torch.distributed.all_gather_into_tensor of out [U, G, d] fp32 ("
                                + ("gloo, ranks sharing one GPU: debug mode, timings meaningless)"
                                   if share_gpu else "NCCL over NVLink)"),
                  "timing": "CUDA events on the launching stream, max over ranks; gather includes the "
                            "pack of the rank's rows"}

    # ---------------- timed region B: the full hot path per layer (rows 1-8), phase events
    full = None
    if not args.skip_full:
        from workload.gen import draw_v0
        calws = torch.zeros(rk.workspace_bytes(
            rk.make_dims(cfg.units, cfg.group, cfg.head_dim, cfg.rank, cfg.n_vis, 0,
                         cfg.q_window, rk.BF16 if cfg.dtype == "bf16" else rk.F32), rk.OP_CALIBRATE),
            dtype=torch.uint8, device=dev)
        V0 = torch.from_numpy(draw_v0(cfg, units=rank_units(cfg, rank))).to(dev)
        n_full = max(2, min(5, args.steps))

        def full_path(calibrate):
            phase_ms = {"calibrate": 0.0, "compress": 0.0, "decode": 0.0}
            for it in range(1 + n_full):
                evs = []
                with torch.cuda.stream(stream):
                    for ly in layers:
                        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                        e[0].record(stream)
                        cal = calibrate(ly)
                        e[1].record(stream)
                        rk.compress_kv(ly["K"], cal["R"], out=ly["Kc"], stream=stream)
                        e[2].record(stream)
                        rk.decode_attn(ly["q"], ly["Kc"], ly["V"], cal["R"], cal["dmu"],
                                       ly["Ktext"], ly["Vtext"], out=ly["out"], ws=ws, stream=stream)
                        e[3].record(stream)
                        evs.append(e)
                torch.cuda.synchronize()
                if it == 0:
                    continue  # warm-up pass
                for e in evs:
                    phase_ms["calibrate"] += e[0].elapsed_time(e[1])
                    phase_ms["compress"] += e[1].elapsed_time(e[2])
                    phase_ms["decode"] += e[2].elapsed_time(e[3])
            per_layer_us = {k: round(1e3 * v / (n_full * L), 2) for k, v in phase_ms.items()}
            cb = compress_bytes(cfg)
            return {"ms_per_step": round(sum(phase_ms.values()) / n_full, 3), "layers": L,
                    "us_per_layer": per_layer_us,
                    "prefill_tokens_per_s": round(cfg.units * cfg.n_vis / (
                        (per_layer_us["calibrate"] + per_layer_us["compress"]) * 1e-6), 1),
                    "compress_gbs_1pass_bytes": round(cb / (per_layer_us["compress"] * 1e-6) / 1e9, 1)}

        full = {"solver": "one-sided Jacobi on a pivoted-Cholesky factor (fp32, registers) + fp64 refinement of the r + 8 leading columns on DMMA (north_star; eigh arm P:653)"}
        full.update(full_path(lambda ly: rk.calibrate(ly["K"], ly["Qw"], cfg.rank, ws=calws,
                                                      stream=stream)))
        sub = {"solver": "Cholesky-QR subspace iteration, T=5 (paper default, NEXT-1)"}
        sub.update(full_path(lambda ly: rk.calibrate_subspace(ly["K"], ly["Qw"], V0, ws=calws,
                                                              stream=stream)))
        full["subspace_solver"] = sub

    # ---------------- e2e: full path from pinned host buffers, H2D/D2H inside the timed region
    e2e = None
    if not args.skip_e2e:
        names = ("K", "V", "Ktext", "Vtext", "Qw", "q")
        pinned = {k: _to_dev(host[k], dev).cpu().pin_memory() for k in names}
        dbuf = {k: torch.empty_like(pinned[k], device=dev) for k in names}
        out_h = torch.empty((cfg.units, cfg.group, cfg.head_dim), dtype=torch.float32).pin_memory()
        Kc_d = torch.empty_like(layers[0]["Kc"])
        calws2 = torch.zeros(rk.workspace_bytes(
            rk.make_dims(cfg.units, cfg.group, cfg.head_dim, cfg.rank, cfg.n_vis, 0,
                         cfg.q_window, rk.BF16 if cfg.dtype == "bf16" else rk.F32), rk.OP_CALIBRATE),
            dtype=torch.uint8, device=dev)
        h2d = sum(v.numel() * v.element_size() for v in pinned.values())
        d2h = out_h.numel() * 4

        # one copy stream, prefill inputs first: K and Q_W cross PCIe at the full link rate,
        # then the decode inputs (V, text K/V, q) cross while calibrate + compress run on the
        # compute stream (PCIe and the eigensolver overlap); the decode waits for them.  (r1
        # copied K and V concurrently on two streams: K then shared the link with V and the
        # eigensolve started ~12 ms later.)
        copy_stream = torch.cuda.Stream(device=dev)
        ev_k = torch.cuda.Event()
        ev_in = torch.cuda.Event()
        ev_go = torch.cuda.Event()

        def e2e_step():
            ev_go.record(stream)
            copy_stream.wait_event(ev_go)          # previous step's decode is done with dbuf
            with torch.cuda.stream(copy_stream):
                for k in ("K", "Qw"):
                    dbuf[k].copy_(pinned[k], non_blocking=True)
                ev_k.record(copy_stream)
                for k in ("V", "Ktext", "Vtext", "q"):
                    dbuf[k].copy_(pinned[k], non_blocking=True)
                ev_in.record(copy_stream)
            with torch.cuda.stream(stream):
                stream.wait_event(ev_k)
                cal = rk.calibrate(dbuf["K"], dbuf["Qw"], cfg.rank, ws=calws2, stream=stream)
                rk.compress_kv(dbuf["K"], cal["R"], out=Kc_d, stream=stream)
                stream.wait_event(ev_in)
                o = rk.decode_attn(dbuf["q"], Kc_d, dbuf["V"], cal["R"], cal["dmu"],
                                   dbuf["Ktext"], dbuf["Vtext"], ws=ws, stream=stream)
                out_h.copy_(o, non_blocking=True)

        e2e_step()
        barrier()
        n_e2e = max(2, min(5, args.steps))
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        a1.record(stream)
        barrier()
        e_ms = max_ranks(a0.elapsed_time(a1) / n_e2e)
        e2e = {"value": round(world * bytes_layer / (e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(e_ms, 3),
               "path": "pinned host -> H2D (K, Q_W) -> calibrate -> compress -> decode -> D2H; the "
                       "decode inputs' H2D follows K's on the copy stream, overlapping calibrate + "
                       "compress (1 layer)"}

    # ---------------- extra rows (N = 1): the GQA configurations under the same clock
    extra = None
    n_extra_launches = 0
    if world == 1 and not args.skip_extra:
        extra = {}
        del host
        for name in EXTRA_ROWS:
            if name == cfg.name:
                continue
            ecfg = CONFIGS[name]
            eb = decode_bytes(ecfg)
            EL = max(2, min(4, int(600e6 // eb) + 1))
            _, elayers, eg, ebad = prepare_layers(rk, ecfg, EL, list(range(ecfg.units)), dev)
            erun, elaunch, _ = decode_graph(rk, ecfg, elayers, stream, 0, not args.no_graph)
            ms = time_region(erun, args.steps, args.warmup, stream, barrier) / args.steps
            n_extra_launches += args.steps * EL * elaunch
            eus = 1e3 * ms / EL
            ach = eb / (eus * 1e-6) / 1e9
            tr = ncu_traffic(name)
            extra[name] = {"us_per_layer": round(eus, 3), "gbs": round(ach, 1),
                           "frac": round(ach / peak_gbs, 4), "pct_of_8tbs": round(100 * ach / NOMINAL_HBM_GBS, 2),
                           "algorithmic_bytes_per_launch": eb, "layers_timed": EL,
                           "ncu_traffic_ratio": round(tr / eb, 4) if tr else None,
                           "calibrate_info_nonzero": ebad, "host_gen_s": round(eg, 1),
                           "kernel": "decode_ring_kernel (CTA ring, TMA, mma.sync)"}
            del elayers
            torch.cuda.empty_cache()

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.skip_cpu:
        cpu = oracle_baseline(cfg, args.cpu_seconds)

    traffic = ncu_traffic(cfg.name)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": cfg.dtype, "data": "synthetic (seeded nat distribution, SURVEY §8(d))",
        "config": {"workload": cfg.name, "batch_per_gpu": cfg.batch, "global_batch": cfg.batch * world,
                   "h_kv": cfg.h_kv, "group": cfg.group, "units_per_gpu": cfg.units,
                   "head_dim": cfg.head_dim, "rank": cfg.rank, "n_vis": cfg.n_vis,
                   "n_text": cfg.n_text, "layers_timed": L,
                   "parallelism": f"units sharded by (batch x kv head), weak, {world} GPU(s)",
                   "l2": "inputs larger than L2 (decode bytes/layer %.0f MB x %d layers > 126 MB)"
                         % (bytes_layer / 1e6, L),
                   "cuda_graph": not args.no_graph},
        "us_per_layer": round(us_layer, 3),
        "pct_of_8tbs": round(100 * achieved / NOMINAL_HBM_GBS, 2),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak_gbs,
                     "unit": "GB/s", "frac": round(achieved / peak_gbs, 4), "traffic": traffic,
                     "peak_kind": peak_kind,
                     # frac > 1 is possible: the measured peak is a read+write copy, this
                     # kernel is a read-dominated stream (99.7 % reads, ncu)
                     "algorithmic_bytes_per_launch": bytes_layer,
                     # the automatic choice (decode.cu launch_decode): the CTA ring for
                     # G >= 2 and for G = 1 batches of <= 2 units per SM
                     "kernel": ("rotatek decode (decode_fast_kernel: cp.async.bulk warp streaming, "
                                "CUDA cores)" if cfg.group == 1 and cfg.units > 2 * 148 else
                                "rotatek decode (decode_ring_kernel: CTA ring, tensor-map TMA, "
                                "mma.sync)")},
        "decode_tflops": round(decode_flops(cfg) / (us_layer * 1e-6) / 1e12, 3),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "full_step": full,
        "extra_rows": extra,
        "strong": strong,
        "clocks": clocks.summary(),
        "gpu_launches": args.steps * L * launches_per_decode,
        "launches_per_decode": launches_per_decode,
        "extra_rows_launches": n_extra_launches,
        "calibrate_info_nonzero": bad_info,
        "host_gen_s": round(t_gen, 1),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return 0
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        return relaunch(args)
    if world_env is not None and int(world_env) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world_env}"}), flush=True)
        return 2
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
