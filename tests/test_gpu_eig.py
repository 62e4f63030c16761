"""GPU: the eigensolvers behind rotatek_calibrate (step 4) against the fp64 oracle.

The default d = 128 solver is one-sided (Hestenes) Jacobi on a pivoted-Cholesky factor of
C_q with the columns in registers (csrc/hestenes.cu); ROTATEK_EIG_TWOSIDED selects the
two-sided packed-triangle kernel.  Both are followed by the fp64 refinement and must pass the
G-cal gates of tests/test_gpu_parity.py::test_calibrate_gap_data.  The one-sided kernel hands
a unit whose C_q has an exactly null column (a constant or dead key channel) to the two-sided
kernel; rank-deficient C_q (fewer tokens than channels) stays on the one-sided path.
"""
import numpy as np
import pytest

from helpers import mask_bits_u32, to_np64, to_torch
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


def _flags(rk, solver):
    return rk.DEFAULT_FLAGS | (rk.EIG_TWOSIDED if solver == "twosided" else 0)


def _check(cal, ref, r, units, projector=True):
    """G-cal: projector vs the oracle (planted gap only), orthonormal R_r, R_r^T C_q R_r
    diagonal, sum of eigenvalues = trace, captured variance, bit-exact select on the GPU's
    own eigenvalues."""
    R = to_np64(cal["R"])
    lam = to_np64(cal["eigvals"])
    for u in units:
        Cq = ref["Cq"][u]
        nrm = np.linalg.norm(Cq)
        if projector:
            P, Pref = R[u] @ R[u].T, ref["R"][u] @ ref["R"][u].T
            assert np.linalg.norm(P - Pref) <= 1e-3, u
        assert np.linalg.norm(R[u].T @ R[u] - np.eye(r)) <= 1e-3, u
        D = R[u].T @ Cq @ R[u]
        assert np.linalg.norm(D - np.diag(np.diag(D))) / nrm <= 1e-5, u
        assert abs(lam[u].sum() - np.trace(Cq)) <= 1e-5 * abs(np.trace(Cq)) + 1e-6 * nrm, u
        captured = np.trace(D) / np.sort(ref["lam"][u])[-r:].sum()
        assert captured >= 1 - 1e-5, u
        om, oi = orc.select_topr(lam[u], r)
        np.testing.assert_array_equal(cal["idx"][u].cpu().numpy(), oi)
        np.testing.assert_array_equal(mask_bits_u32(cal["mask"][u].cpu().numpy()), om)


@pytest.mark.parametrize("solver", ["onesided", "twosided"])
@pytest.mark.parametrize("dist,mean", [("gap", 0.5), ("gap", 20.0), ("nat", 0.5)])
def test_solver_gates(rk, solver, dist, mean):
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=6, n_vis=500, n_text=0)
    w = make_workload(cfg, dist=dist, mean=mean)
    cal = rk.calibrate(to_torch(w["K"]), to_torch(w["Qw"]), cfg.rank, _flags(rk, solver), want_full=True)
    torch.cuda.synchronize()
    ref = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    assert (cal["info"].cpu().numpy() == 0).all()
    # natural keys have no planted gap at r: subspace-invariant gates only
    _check(cal, ref, cfg.rank, range(cfg.units), projector=dist == "gap")
    Rf = to_np64(cal["R_full"])  # the full basis is orthonormal too (clusters included)
    for u in range(cfg.units):
        assert np.linalg.norm(Rf[u].T @ Rf[u] - np.eye(cfg.head_dim)) <= 1e-3, u


def test_solvers_agree_full_size(rk):
    """llava_b32 (1024 units, the bench launch): one-sided vs two-sided top-r projectors."""
    import torch
    cfg = CONFIGS["llava_b32"]
    w = make_workload(cfg, threads=16)
    K, Qw = to_torch(w["K"]), to_torch(w["Qw"])
    a = rk.calibrate(K, Qw, cfg.rank, _flags(rk, "onesided"))
    b = rk.calibrate(K, Qw, cfg.rank, _flags(rk, "twosided"))
    torch.cuda.synchronize()
    assert (a["info"] == 0).all() and (b["info"] == 0).all()
    Ra, Rb = a["R"].double(), b["R"].double()
    dP = torch.linalg.matrix_norm(Ra @ Ra.transpose(1, 2) - Rb @ Rb.transpose(1, 2))
    assert dP.max().item() <= 1e-3
    # sampled units against the oracle (projector distance is meaningful where the oracle's
    # r-th and (r+1)-th eigenvalues separate; the e2e gates live in test_gpu_parity.py)
    sample = [0, 411, 1023]
    sub = make_workload(cfg, units=sample)
    ref = orc.calibrate(sub["K"].f64(), sub["Qw"].f64(), cfg.rank)
    Ra_np = to_np64(a["R"][sample])
    for j in range(len(sample)):
        lam = np.sort(ref["lam"][j])[::-1]
        rel_gap = (lam[cfg.rank - 1] - lam[cfg.rank]) / lam[0]
        P, Pref = Ra_np[j] @ Ra_np[j].T, ref["R"][j] @ ref["R"][j].T
        assert np.linalg.norm(P - Pref) <= max(1e-3, 1e-8 / rel_gap), (sample[j], rel_gap)


@pytest.mark.parametrize("solver", ["onesided", "twosided"])
def test_null_columns(rk, solver):
    """A constant key channel (unit 1) and two dead channels (unit 2) make C_q's row and column
    exactly zero: the one-sided solver marks the unit and the two-sided kernel re-solves it;
    info ends 0 and every gate holds (the zero eigenvalues sit below the kept r)."""
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=3, n_vis=300, n_text=0)
    w = make_workload(cfg, dist="gap")
    K = to_torch(w["K"]).clone()
    K[1, :, 7] = 1.25
    K[2, :, 3] = 0.0
    K[2, :, 90] = 0.0
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, _flags(rk, solver), want_full=True)
    torch.cuda.synchronize()
    ref = orc.calibrate(to_np64(K), w["Qw"].f64(), cfg.rank)
    assert (cal["info"].cpu().numpy() == 0).all()
    _check(cal, ref, cfg.rank, range(cfg.units))
    Rf = to_np64(cal["R_full"])
    # the full basis stays orthonormal through the fallback; with the default solver a unit
    # re-solved by the two-sided kernel keeps its fp32 basis outside the r + 8 refined
    # columns (rotatek.h, R_full)
    tol = 1e-3 if solver == "twosided" else 5e-3
    for u in range(cfg.units):
        assert np.linalg.norm(Rf[u].T @ Rf[u] - np.eye(cfg.head_dim)) <= tol, u


@pytest.mark.parametrize("solver", ["onesided", "twosided"])
def test_rank_deficient(rk, solver):
    """N = 40 tokens < d = 128: C_q has rank <= 39; the pivoted Cholesky stops early and the
    remaining Schur-complement columns ride along; the top-r = 32 subspace (planted gap) and
    all gates hold."""
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=4, n_vis=40, n_text=0)
    w = make_workload(cfg, dist="gap")
    cal = rk.calibrate(to_torch(w["K"]), to_torch(w["Qw"]), cfg.rank, _flags(rk, solver), want_full=True)
    torch.cuda.synchronize()
    ref = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    assert (cal["info"].cpu().numpy() == 0).all()
    _check(cal, ref, cfg.rank, range(cfg.units))


@pytest.mark.parametrize("solver,fp64", [("onesided", False), ("twosided", False), ("onesided", True)])
def test_nonconvergence_reported(rk, solver, fp64, monkeypatch):
    """Fault injection (SURVEY §5 failure detection): ROTATEK_JACOBI_MAX_SWEEPS=1 caps every
    Jacobi solver at one sweep; info reports the sweeps done (> 0) for every unit and the
    outputs are still written (finite).  The cap is read at every call: lifting it restores
    info 0."""
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=3, n_vis=300, n_text=0)
    w = make_workload(cfg, dist="gap")
    K, Qw = to_torch(w["K"]), to_torch(w["Qw"])
    flags = _flags(rk, solver) | (rk.EIG_FP64 if fp64 else 0)
    monkeypatch.setenv("ROTATEK_JACOBI_MAX_SWEEPS", "1")
    cal = rk.calibrate(K, Qw, cfg.rank, flags)
    torch.cuda.synchronize()
    assert cal["info"].cpu().tolist() == [1] * cfg.units
    assert torch.isfinite(cal["R"]).all() and torch.isfinite(cal["dmu"]).all()
    assert ((cal["idx"] >= 0) & (cal["idx"] < cfg.head_dim)).all()
    monkeypatch.delenv("ROTATEK_JACOBI_MAX_SWEEPS")
    cal = rk.calibrate(K, Qw, cfg.rank, flags)
    torch.cuda.synchronize()
    assert (cal["info"].cpu().numpy() == 0).all()


@pytest.mark.parametrize("rank", [8, 64, 100, 128])
def test_refinement_paths(rank, rk):
    """The fp64 refinement behind the one-sided solver takes the DMMA candidate kernel for
    r + 8 <= 72 (KC = 40 / 72) and the all-column kernel above; planted gap at r, G-cal gates
    (r = d = 128: every column kept, R_r is the full basis)."""
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=3, n_vis=400, n_text=0, rank=rank)
    w = make_workload(cfg, dist="gap")
    cal = rk.calibrate(to_torch(w["K"]), to_torch(w["Qw"]), cfg.rank, want_full=True)
    torch.cuda.synchronize()
    ref = orc.calibrate(w["K"].f64(), w["Qw"].f64(), cfg.rank)
    assert (cal["info"].cpu().numpy() == 0).all()
    _check(cal, ref, cfg.rank, range(cfg.units), projector=rank < cfg.head_dim)


@pytest.mark.parametrize("solver", ["onesided", "twosided"])
def test_wide_spectrum(rk, solver):
    """Keys whose last 64 channels are scaled by 1e-4 (C_q eigenvalues spanning ~1e-8 of the
    largest): the pivoted Cholesky stops at its d eps threshold and the tiny Schur-complement
    columns ride along; the top-r subspace (planted gap) and every gate still hold."""
    import torch
    cfg = CONFIGS["llava_b1"].with_(h_kv=3, n_vis=500, n_text=0)
    w = make_workload(cfg, dist="gap")
    K = to_torch(w["K"]).float()
    K[:, :, 64:] *= 1e-4
    K = K.to(torch.bfloat16).contiguous()
    cal = rk.calibrate(K, to_torch(w["Qw"]), cfg.rank, _flags(rk, solver), want_full=True)
    torch.cuda.synchronize()
    ref = orc.calibrate(to_np64(K), w["Qw"].f64(), cfg.rank)
    assert (cal["info"].cpu().numpy() == 0).all()
    _check(cal, ref, cfg.rank, range(cfg.units), projector=False)
    R = to_np64(cal["R"])
    for u in range(cfg.units):  # the kept subspace = the oracle's wherever its gap is clear
        lam = np.sort(ref["lam"][u])[::-1]
        rel_gap = (lam[cfg.rank - 1] - lam[cfg.rank]) / lam[0]
        P, Pref = R[u] @ R[u].T, ref["R"][u] @ ref["R"][u].T
        assert np.linalg.norm(P - Pref) <= max(1e-3, 1e-7 / rel_gap), (u, rel_gap)
