"""World-size-2 gloo tests of the N > 1 host path (CPU only).

Each rank takes its unit shard exactly as bench.py does, computes its units (the fp64
oracle stands in for the GPU kernel here), and the gathered result must equal the
single-process result bit for bit (units are independent).  The max-over-ranks timing
reduction is checked too.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_19218_b200.sharding import max_over_ranks, strong_units, weak_units


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from workload import CONFIGS, make_workload
        cfg = CONFIGS["llava_b1"].with_(h_kv=6, n_vis=96, n_text=8, head_dim=32, rank=8)
        if mode == "weak":
            units = list(weak_units(cfg.units, rank))
            gcfg = cfg.with_(batch=world)
        else:
            units = list(strong_units(cfg.units, rank, world))
            gcfg = cfg
        w = make_workload(gcfg, units=units, seed=7)
        out = orc.pipeline(w["K"].f64(), w["V"].f64(), w["Qw"].f64(), w["q"].f64(), cfg.rank,
                           "bf16", w["Ktext"].f64(), w["Vtext"].f64())["out"]
        t = torch.from_numpy(np.ascontiguousarray(out))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([t.shape[0]]))
        maxn = int(max(s.item() for s in sizes))
        pad = torch.zeros((maxn,) + tuple(t.shape[1:]), dtype=t.dtype)
        pad[: t.shape[0]] = t
        bufs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        gathered = torch.cat([b[: int(s.item())] for b, s in zip(bufs, sizes)]).numpy()
        mx = max_over_ranks(1.5 + rank)
        if rank == 0:
            full = make_workload(gcfg, seed=7)
            ref = orc.pipeline(full["K"].f64(), full["V"].f64(), full["Qw"].f64(),
                               full["q"].f64(), cfg.rank, "bf16", full["Ktext"].f64(),
                               full["Vtext"].f64())["out"]
            q.put((np.array_equal(gathered, ref), mx, gathered.shape[0]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["weak", "strong"])
def test_two_rank_shards_reproduce_single_process(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    equal, mx, n = q.get(timeout=10)
    assert equal
    assert mx == 2.5
    assert n == (12 if mode == "weak" else 6)


def test_strong_units_cover_exactly():
    for total in (1, 5, 32, 1024):
        for world in (1, 2, 3, 8):
            got = [u for r in range(world) for u in strong_units(total, r, world)]
            assert got == list(range(total))
    assert list(weak_units(4, 3)) == [12, 13, 14, 15]


def _token_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2605_19218_b200.sharding import token_slice
        rng = np.random.default_rng(11)       # every rank draws the same replicated inputs
        U, G, d, r, N, M = 2, 3, 16, 4, 37, 6
        qv = rng.standard_normal((U, G, d))
        Kt = rng.standard_normal((U, N, r))
        V = rng.standard_normal((U, N, d))
        R = np.linalg.qr(rng.standard_normal((U, d, d)))[0][:, :, :r]
        dmu = rng.standard_normal((U, d))
        Kx = rng.standard_normal((U, M, d))
        Vx = rng.standard_normal((U, M, d))
        vs, xs = token_slice(N, world, rank), token_slice(M, world, rank)
        part = orc.decode_partial(qv, Kt[:, vs.start:vs.stop], V[:, vs.start:vs.stop], R, dmu,
                                  Kx[:, xs.start:xs.stop], Vx[:, xs.start:xs.stop])
        t = torch.from_numpy(np.ascontiguousarray(part))
        parts = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype)
        dist.all_gather_into_tensor(parts, t)
        parts = parts.view((world,) + tuple(t.shape))
        if rank == 0:
            out = orc.merge_partials(parts.numpy())
            ref = orc.decode(qv, Kt, V, R, dmu, Kx, Vx)
            q.put(float(np.abs(out - ref).max()))
    finally:
        dist.destroy_process_group()


def test_two_rank_token_shards_merge_to_full_decode():
    """Token sharding for U < P: each rank's Alg. 2 state over its token
    slice, all-gathered and merged, equals the unsharded decode (exact re-association)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_token_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get(timeout=10) <= 1e-12


def test_token_slices_cover_exactly():
    from paper_2605_19218_b200.sharding import token_slice
    for n in (1, 7, 64, 2880):
        for world in (1, 2, 3, 8):
            got = [t for r in range(world) for t in token_slice(n, world, r)]
            assert got == list(range(n))
