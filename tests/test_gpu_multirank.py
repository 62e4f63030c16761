"""World-size-2 runs of the PRODUCT sharding functions on the CUDA path.

The round's boxes have one GPU, so both ranks share cuda:0 and the collective is gloo
(sharding._all_gather stages device rows through the host; with NCCL it is one
all_gather_into_tensor over NVLink).  Every rank calibrates, compresses and decodes through
librotatek's kernels:
  * unit sharding (strong scaling of a fixed batch): sharding.decode_unit_sharded on the
    rank's unit range, outputs gathered, equals the single-process decode of the whole
    batch (to fp32 re-association: the kernels split a unit's tokens over CTAs according to
    the batch they see) and the oracle (G-dec on the GPU's cache bytes);
  * token sharding (U < P): sharding.decode_token_sharded on the rank's contiguous slice of
    every unit's visual and text tokens, states gathered and merged by the merge kernel.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, here)
        sys.path.insert(0, os.path.dirname(here))
        from helpers import max_rel_err, to_np64, to_torch
        from oracle import oracle as orc
        import paper_2605_19218_b200 as rk
        from paper_2605_19218_b200.sharding import (decode_token_sharded, decode_unit_sharded,
                                                    strong_units, token_slice)
        from workload import CONFIGS, make_workload
        torch.cuda.set_device(0)
        cfgs = {"llava": CONFIGS["llava_b1"].with_(h_kv=5, n_vis=700, n_text=33),
                "qwen": CONFIGS["qwen_b1_r32"].with_(h_kv=3, n_vis=900, n_text=20)}
        cfg = cfgs[name]
        w = make_workload(cfg, seed=21)
        K = to_torch(w["K"])
        cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank)
        Kc = rk.compress_kv(K, cal["R"])
        args = [to_torch(w["q"]), Kc, to_torch(w["V"]), cal["R"], cal["dmu"],
                to_torch(w["Ktext"]), to_torch(w["Vtext"])]
        full = rk.decode_attn(*args)
        if mode == "units":
            rng = strong_units(cfg.units, rank, world)
            mine = [a[rng.start:rng.stop].contiguous() for a in args]
            got = decode_unit_sharded(*mine, total_units=cfg.units)
        else:
            vs, xs = token_slice(cfg.n_vis, world, rank), token_slice(cfg.n_text, world, rank)
            q_, Kc_, V_, R_, dmu_, Kt_, Vt_ = args
            got = decode_token_sharded(q_, Kc_[:, vs.start:vs.stop].contiguous(),
                                       V_[:, vs.start:vs.stop].contiguous(), R_, dmu_,
                                       Kt_[:, xs.start:xs.stop].contiguous(),
                                       Vt_[:, xs.start:xs.stop].contiguous())
        torch.cuda.synchronize()
        if rank == 0:
            ref = orc.decode(w["q"].f64(), to_np64(Kc), w["V"].f64(), to_np64(cal["R"]), to_np64(cal["dmu"]),
                             w["Ktext"].f64(), w["Vtext"].f64())
            q.put((tuple(got.shape), max_rel_err(to_np64(got), to_np64(full)), max_rel_err(to_np64(got), ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["units", "tokens"])
@pytest.mark.parametrize("name", ["llava", "qwen"])
def test_two_rank_product_sharding_on_gpu(name, mode):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    shape, err_full, err_orc = q.get(timeout=10)
    assert shape[0] == (5 if name == "llava" else 3)
    assert err_full <= 1e-5, err_full      # fp32 re-association only
    assert err_orc <= 2e-3, err_orc         # G-dec on the GPU's cache bytes
