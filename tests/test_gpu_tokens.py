"""GPU parity of the token-selection prefill (NEXT-2; reading Q20) against
the oracle on the selected tokens.

rotatek_calibrate_tokens / rotatek_compress_kv_tokens gather each unit's surviving key rows
(a FastV/VisionZip-style sorted subset of an unpruned cache, or the first n_u rows of a padded
batch) inside the tensor-core producers.  The oracle gets the SELECTED rows as plain arrays
(numpy fancy indexing, unit by unit), so a kernel that folded padding or unselected rows into
mu / C_q, or gathered the wrong rows, fails the projector / output comparisons.
"""
import numpy as np
import pytest

from helpers import max_rel_err, to_np64, to_torch
from oracle import oracle as orc
from workload import CONFIGS, make_workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    import torch
    assert torch.cuda.is_available()
    import paper_2605_19218_b200 as rk
    rk.lib()
    return rk


CASES = {
    "llava": CONFIGS["llava_b1"].with_(h_kv=4, n_vis=600, n_text=17),
    "qwen": CONFIGS["qwen_b1_r32"].with_(h_kv=3, n_vis=900, n_text=9),
    "qwen_r64": CONFIGS["qwen_b1_r32"].with_(h_kv=2, rank=64, n_vis=700, n_text=0),
}


def _per_unit_ref(cfg, K, V, Qw, q, Kx, Vx, rows):
    """Oracle steps 1-8 per unit on the selected key / value rows (rows[u]: int array)."""
    outs, Rs = [], []
    for u in range(cfg.units):
        sel = rows[u]
        ref = orc.pipeline(K[u:u + 1, sel], V[u:u + 1, sel], Qw[u:u + 1], q[u:u + 1], cfg.rank, "bf16",
                           Kx[u:u + 1] if Kx is not None else None, Vx[u:u + 1] if Vx is not None else None)
        outs.append(ref["out"][0])
        Rs.append(ref["R"][0])
    return np.stack(outs), Rs


@pytest.mark.parametrize("name", list(CASES))
def test_token_list_prefill(rk, name):
    """Calibrate + compress on a sorted random 30 % subset of each unit's rows (the joint
    config's FastV-style survivors), decode on the compressed survivors; equals the
    oracle run on the survivors only.  The unselected rows carry huge values, so any of them
    leaking into the covariance would change the rotation."""
    import torch
    cfg = CASES[name]
    w = make_workload(cfg)
    M = cfg.n_text
    rng = np.random.default_rng(5)
    n_keep = int(round(0.30 * cfg.n_vis))
    rows = [np.sort(rng.choice(cfg.n_vis, n_keep, replace=False)) for _ in range(cfg.units)]
    K = to_torch(w["K"]).clone()
    junk = torch.ones(K.shape, dtype=torch.bool, device="cuda")
    for u in range(cfg.units):
        junk[u, torch.from_numpy(rows[u]).cuda()] = False
    K[junk] = 300.0
    idx = torch.from_numpy(np.stack(rows).astype(np.int32)).cuda()
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, tok_idx=idx)
    Kc = rk.compress_kv(K, cal["R"], tok_idx=idx)
    V = to_torch(w["V"])
    Vs = torch.stack([V[u, idx[u].long()] for u in range(cfg.units)]).contiguous()
    out = rk.decode_attn(to_torch(w["q"]), Kc, Vs, cal["R"], cal["dmu"],
                         to_torch(w["Ktext"]) if M else None, to_torch(w["Vtext"]) if M else None)
    torch.cuda.synchronize()
    assert (cal["info"].cpu().numpy() == 0).all()
    assert Kc.shape == (cfg.units, n_keep, cfg.rank)
    ref, _ = _per_unit_ref(cfg, w["K"].f64(), w["V"].f64(), w["Qw"].f64(), w["q"].f64(),
                           w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None, rows)
    assert max_rel_err(to_np64(out), ref) <= 2e-3
    # the fused gather equals calibrate / compress on an explicitly compacted K, bit for bit
    Kg = torch.stack([K[u, idx[u].long()] for u in range(cfg.units)]).contiguous()
    cal2 = rk.calibrate(Kg, to_torch(w["Qw"]), cfg.rank)
    Kc2 = rk.compress_kv(Kg, cal2["R"])
    torch.cuda.synchronize()
    assert torch.equal(cal["R"], cal2["R"]) and torch.equal(Kc, Kc2)


@pytest.mark.parametrize("name", list(CASES))
def test_per_unit_lengths_prefill(rk, name):
    """A padded batch of requests with different image-token counts: unit u has n_u valid rows
    (padding rows hold garbage, even NaN).  Calibrate / compress with n_vis_u, decode with the
    same lengths (rotatek_decode_attn_varlen); each unit equals the oracle on its first n_u
    rows, and K~ rows past n_u are exactly 0."""
    import torch
    cfg = CASES[name]
    w = make_workload(cfg)
    M = cfg.n_text
    rng = np.random.default_rng(9)
    nv = rng.integers(cfg.rank + 2, cfg.n_vis + 1, cfg.units).astype(np.int32)
    nv[0] = cfg.n_vis
    K = to_torch(w["K"]).clone()
    for u in range(cfg.units):
        K[u, int(nv[u]):] = float("nan")
    lens = torch.from_numpy(nv).cuda()
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, n_vis_u=lens)
    Kc = rk.compress_kv(K, cal["R"], n_vis_u=lens)
    out = rk.decode_attn(to_torch(w["q"]), Kc, to_torch(w["V"]), cal["R"], cal["dmu"],
                         to_torch(w["Ktext"]) if M else None, to_torch(w["Vtext"]) if M else None,
                         n_vis_u=lens)
    torch.cuda.synchronize()
    assert (cal["info"].cpu().numpy() == 0).all()
    for u in range(cfg.units):
        assert (Kc[u, int(nv[u]):] == 0).all()
    rows = [np.arange(int(n)) for n in nv]
    ref, _ = _per_unit_ref(cfg, w["K"].f64(), w["V"].f64(), w["Qw"].f64(), w["q"].f64(),
                           w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None, rows)
    assert max_rel_err(to_np64(out), ref) <= 2e-3


def test_joint_config_from_mask(rk):
    """Config 4 (joint token-channel pruning, LLaVA shape, b = 64) straight from the token
    mask: the 864 FastV-style survivors of each unit's 2880-position cache are gathered by the
    prefill kernels (no compacted K), sampled units checked against the oracle."""
    import torch
    cfg = CONFIGS["joint_b64"]
    full = cfg.with_(n_vis=cfg.n_vis_full, n_vis_full=0)
    sample = [0, 1000, 2047]
    w = make_workload(full, threads=16)
    rng = np.random.default_rng(2)
    rows = np.stack([np.sort(rng.choice(full.n_vis, cfg.n_vis, replace=False)) for _ in range(cfg.units)])
    idx = torch.from_numpy(rows.astype(np.int32)).cuda()
    K = to_torch(w["K"])
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, tok_idx=idx)
    Kc = rk.compress_kv(K, cal["R"], tok_idx=idx)
    V = rk.gather_tokens(to_torch(w["V"]), idx)   # V is read once at decode: compact it once
    out = rk.decode_attn(to_torch(w["q"]), Kc, V, cal["R"], cal["dmu"], to_torch(w["Ktext"]),
                         to_torch(w["Vtext"]))
    torch.cuda.synchronize()
    sub = make_workload(full, units=sample)
    sel = [rows[u] for u in sample]
    scfg = cfg.with_(batch=1, h_kv=len(sample))
    ref, _ = _per_unit_ref(scfg, sub["K"].f64(), sub["V"].f64(), sub["Qw"].f64(), sub["q"].f64(),
                           sub["Ktext"].f64(), sub["Vtext"].f64(), sel)
    assert max_rel_err(to_np64(out[sample]), ref) <= 2e-3
