"""GPU parity of the subspace-iteration solver (NEXT-1) against the fp64 oracle."""
import numpy as np
import pytest

from helpers import max_rel_err, to_np64, to_torch
from oracle import oracle as orc
from workload import CONFIGS, make_workload
from workload.gen import draw_v0

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rk():
    import torch
    assert torch.cuda.is_available()
    import paper_2605_19218_b200 as rk
    rk.lib()
    return rk


@pytest.mark.parametrize("name,cfg", [
    ("llava_small", CONFIGS["llava_b1"].with_(h_kv=3, n_vis=500, n_text=17)),
    ("qwen_small", CONFIGS["qwen_b1_r32"].with_(h_kv=2, n_vis=700, n_text=9)),
    ("qwen_r64", CONFIGS["qwen_b1_r32"].with_(h_kv=2, rank=64, n_vis=400, n_text=0)),
    ("toy", CONFIGS["toy"].with_(n_text=3)),
])
@pytest.mark.parametrize("dist", ["nat", "gap"])
def test_subspace_matches_oracle(rk, name, cfg, dist):
    import torch
    w = make_workload(cfg, dist=dist)
    V0 = draw_v0(cfg)
    K = to_torch(w["K"])
    cal = rk.calibrate_subspace(K, to_torch(w["Qw"]), torch.from_numpy(V0).cuda())
    torch.cuda.synchronize()
    assert (cal["info"].cpu().numpy() == 0).all()
    ref = orc.calibrate_subspace(w["K"].f64(), w["Qw"].f64(), V0)
    R = to_np64(cal["R"])
    # same start basis and arithmetic order up to rounding: compare the bases themselves
    scale = np.abs(ref["R"]).max()
    assert np.abs(R - ref["R"]).max() <= 2e-4 * scale, np.abs(R - ref["R"]).max()
    # delta_mu from the stored R
    np.testing.assert_allclose(to_np64(cal["dmu"]), orc.dmu_from_R(R, ref["mu"]), atol=2e-5, rtol=1e-5)
    # Rayleigh quotients
    ritz = np.einsum("uij,uik,ukj->uj", R, ref["Cq"], R) / np.einsum("uij,uij->uj", R, R)
    np.testing.assert_allclose(to_np64(cal["ritz"]), ritz, rtol=1e-4)
    # compress + decode on the GPU's stored basis against oracle steps 7-8 "as stored"
    # (K~ = RNE(K R_gpu), delta_mu from R_gpu): the basis itself is compared above
    M = cfg.n_text
    Kc = rk.compress_kv(K, cal["R"])
    out = rk.decode_attn(to_torch(w["q"]), Kc, to_torch(w["V"]), cal["R"], cal["dmu"],
                         to_torch(w["Ktext"]) if M else None, to_torch(w["Vtext"]) if M else None)
    torch.cuda.synchronize()
    Kt = orc.quantize(orc.compress(w["K"].f64(), R), "bf16")
    want = orc.decode(w["q"].f64(), Kt, w["V"].f64(), R, orc.dmu_from_R(R, ref["mu"]),
                      w["Ktext"].f64() if M else None, w["Vtext"].f64() if M else None)
    assert max_rel_err(to_np64(out), want) <= 2e-3


def test_subspace_gap_data_reaches_eigenspace(rk):
    """App. D parity: with lambda_r / lambda_{r+1} >~ 30 (planted gap), T = 5 lands on the
    exact top-r eigenspace of the oracle's Jacobi."""
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=4, n_vis=900, n_text=0)
    w = make_workload(cfg, dist="gap")
    V0 = draw_v0(cfg)
    cal = rk.calibrate_subspace(to_torch(w["K"]), to_torch(w["Qw"]), torch.from_numpy(V0).cuda())
    torch.cuda.synchronize()
    ref = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    R = to_np64(cal["R"])
    for u in range(cfg.units):
        P = R[u] @ np.linalg.solve(R[u].T @ R[u], R[u].T)
        Pr = ref["R"][u] @ ref["R"][u].T
        assert np.linalg.norm(P - Pr) < 1e-3
