"""GPU parity of the calibration MODES against the fp64 oracle, through the C ABI.

The paper's default (Alg. 1 l.1-5) is the centered, query-weighted covariance
C_q = (sigma sigma^T) . (K - mu)^T (K - mu).  The ABI also exposes
  * ROTATEK_CENTER off            -> mu = 0, C = K^T K: north_star's literal "Key covariance
                                     K^T K" (reading N1/Q2); delta_mu = 0;
  * ROTATEK_QUERY_WEIGHT off, or q_window W = 0 (Qw = NULL)
                                  -> sigma == 1: the "Q-agnostic (K-only PCA)" arm of the
                                     paper's ablation (tab:rotatek-ablation);
and both solvers (Jacobi eigendecomposition, subspace iteration, NEXT-1).  Every mode is
compared with the oracle run in the same mode (oracle.calibrate / calibrate_subspace /
pipeline with center= / query_weight=): projectors on planted-gap data, eigen invariants,
delta_mu, and end-to-end outputs at small sizes and sampled at full size.
"""
import numpy as np
import pytest

from helpers import max_rel_err, to_np64, to_torch
from oracle import oracle as orc
from workload import CONFIGS, make_workload
from workload.gen import draw_v0

pytestmark = pytest.mark.gpu

TOL = {"bf16": 2e-3, "f32": 1e-5}
MODES = {  # name: (center, query_weight, pass Qw)
    "uncentered": (False, True, True),
    "q_agnostic": (True, False, True),
    "uncentered_q_agnostic": (False, False, True),
    "window_0": (True, False, False),  # W = 0: sigma == 1 without the flag
}


@pytest.fixture(scope="module")
def rk():
    import torch
    assert torch.cuda.is_available()
    import paper_2605_19218_b200 as rk
    rk.lib()
    return rk


def _flags(rk, center, qw):
    return (rk.CENTER if center else 0) | (rk.QUERY_WEIGHT if qw else 0)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_calibrate_mode_gap_data(rk, mode, dtype):
    """G-cal in each mode: planted gap (lambda_r / lambda_r+1 ~ 200), so the top-r
    subspace is well defined; projector, orthonormality, diagonalisation of the mode's C_q,
    trace identity, captured variance, and delta_mu from the stored R (zero uncentered)."""
    import torch
    center, qw, pass_qw = MODES[mode]
    cfg = CONFIGS["llava_b1"].with_(h_kv=4, n_vis=777, n_text=0, dtype=dtype)
    w = make_workload(cfg, dist="gap", mean=3.0)
    K = to_torch(w["K"])
    cal = rk.calibrate(K, to_torch(w["Qw"]) if pass_qw else None, cfg.rank, _flags(rk, center, qw))
    torch.cuda.synchronize()
    ref = orc.calibrate(w["K"].f64(), w["Qw"].f64() if pass_qw else None, cfg.rank, center=center,
                        query_weight=qw and pass_qw)
    assert (cal["info"].cpu().numpy() == 0).all()
    R = to_np64(cal["R"])
    lam = to_np64(cal["eigvals"])
    for u in range(cfg.units):
        P, Pref = R[u] @ R[u].T, ref["R"][u] @ ref["R"][u].T
        assert np.linalg.norm(P - Pref) <= 1e-3, (mode, u)
        assert np.linalg.norm(R[u].T @ R[u] - np.eye(cfg.rank)) <= 1e-3
        Cq = ref["Cq"][u]
        nrm = np.linalg.norm(Cq)
        D = R[u].T @ Cq @ R[u]
        assert np.linalg.norm(D - np.diag(np.diag(D))) / nrm <= 1e-5
        assert abs(lam[u].sum() - np.trace(Cq)) <= 1e-5 * abs(np.trace(Cq)) + 1e-6 * nrm
        assert np.trace(D) / np.sort(ref["lam"][u])[-cfg.rank:].sum() >= 1 - 1e-5
    if center:
        np.testing.assert_allclose(to_np64(cal["dmu"]), orc.dmu_from_R(R, ref["mu"]), atol=1e-4, rtol=1e-5)
    else:
        assert (cal["dmu"] == 0).all()   # mu = 0 => delta_mu = 0 (header: zeros if !CENTER)
        assert np.abs(ref["mu"]).max() == 0


E2E = {
    "llava_small": CONFIGS["llava_b1"].with_(h_kv=3, n_vis=333, n_text=37),
    "qwen_small": CONFIGS["qwen_b1_r32"].with_(h_kv=2, n_vis=517, n_text=21),
    "qwen_small_r64": CONFIGS["qwen_b1_r32"].with_(h_kv=2, rank=64, n_vis=300, n_text=12),
}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("name", list(E2E))
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_end_to_end_mode(rk, mode, name, dtype):
    """G-e2e in each mode: calibrate (flags) -> compress -> decode on the GPU against oracle
    steps 1-8 in the same mode, on the natural (outlier-channel, RoPE) distribution."""
    import torch
    center, qw, pass_qw = MODES[mode]
    cfg = E2E[name].with_(dtype=dtype)
    w = make_workload(cfg)
    M = cfg.n_text
    K = to_torch(w["K"])
    cal = rk.calibrate(K, to_torch(w["Qw"]) if pass_qw else None, cfg.rank, _flags(rk, center, qw))
    Kc = rk.compress_kv(K, cal["R"])
    out = rk.decode_attn(to_torch(w["q"]), Kc, to_torch(w["V"]), cal["R"], cal["dmu"],
                         to_torch(w["Ktext"]) if M else None, to_torch(w["Vtext"]) if M else None)
    torch.cuda.synchronize()
    ref = orc.pipeline(w["K"].f64(), w["V"].f64(), w["Qw"].f64() if pass_qw else None, w["q"].f64(),
                       cfg.rank, dtype, w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None,
                       center=center, query_weight=qw and pass_qw)
    err = max_rel_err(to_np64(out), ref["out"])
    assert err <= TOL[dtype], (mode, name, dtype, err)


@pytest.mark.parametrize("mode", ["uncentered", "q_agnostic"])
def test_full_size_sampled_mode(rk, mode):
    """BASELINE.json's LLaVA-NeXT-7B shape at full size (b = 32, 1024 units) in the uncentered
    (north_star's literal K^T K) and query-agnostic modes: sampled units recomputed by the
    oracle one by one from the same seeded bytes."""
    import torch
    center, qw, _ = MODES[mode]
    cfg = CONFIGS["llava_b32"]
    sample = [0, 433, 1023]
    w = make_workload(cfg, threads=16)
    K = to_torch(w["K"])
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, _flags(rk, center, qw))
    Kc = rk.compress_kv(K, cal["R"])
    out = rk.decode_attn(to_torch(w["q"]), Kc, to_torch(w["V"]), cal["R"], cal["dmu"],
                         to_torch(w["Ktext"]), to_torch(w["Vtext"]))
    torch.cuda.synchronize()
    assert (cal["info"].cpu().numpy() >= 0).all()
    sub = make_workload(cfg, units=sample)
    ref = orc.pipeline(sub["K"].f64(), sub["V"].f64(), sub["Qw"].f64(), sub["q"].f64(), cfg.rank, "bf16",
                       sub["Ktext"].f64(), sub["Vtext"].f64(), center=center, query_weight=qw)
    assert max_rel_err(to_np64(out[sample]), ref["out"]) <= 2e-3


@pytest.mark.parametrize("mode", ["uncentered", "q_agnostic", "window_0"])
def test_subspace_mode(rk, mode):
    """The subspace-iteration solver (NEXT-1) in each mode against oracle.calibrate_subspace
    with the same V0 and mode: same start basis and arithmetic order up to rounding, so the
    bases themselves are compared; delta_mu from the stored R."""
    import torch
    center, qw, pass_qw = MODES[mode]
    cfg = CONFIGS["qwen_b1_r32"].with_(h_kv=2, n_vis=700, n_text=0)
    w = make_workload(cfg)
    V0 = draw_v0(cfg)
    K = to_torch(w["K"])
    cal = rk.calibrate_subspace(K, to_torch(w["Qw"]) if pass_qw else None, torch.from_numpy(V0).cuda(),
                                flags=_flags(rk, center, qw))
    torch.cuda.synchronize()
    assert (cal["info"].cpu().numpy() == 0).all()
    ref = orc.calibrate_subspace(w["K"].f64(), w["Qw"].f64() if pass_qw else None, V0, center=center,
                                 query_weight=qw and pass_qw)
    R = to_np64(cal["R"])
    scale = np.abs(ref["R"]).max()
    assert np.abs(R - ref["R"]).max() <= 2e-4 * scale
    if center:
        np.testing.assert_allclose(to_np64(cal["dmu"]), orc.dmu_from_R(R, ref["mu"]), atol=2e-5, rtol=1e-5)
    else:
        assert (cal["dmu"] == 0).all()
