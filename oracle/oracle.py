"""fp64 CPU oracle for the RotateK hot path -- ctypes wrapper around oracle.c.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  It shares no code with the CUDA path (``paper_2605_19218_b200``) and
imports nothing from it.

Every function follows a numbered step of the paper's Alg. 1 / Alg. 2
(PAPER.md P:940-1012); see the per-function citations in ``oracle.c``.
Inputs are numpy arrays of any float dtype; they are converted to fp64
(exactly, for bf16/fp32 values) before the C code runs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

JACOBI_TOL = 1e-13      # reading Q24: off(A) <= 1e-13 ||A||_F
JACOBI_MAX_SWEEPS = 100


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (plain -O2, OpenMP over units)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            path = build()
            L = ctypes.CDLL(path)
            dp = ctypes.POINTER(ctypes.c_double)
            up = ctypes.POINTER(ctypes.c_uint32)
            ip = ctypes.POINTER(ctypes.c_int32)
            i = ctypes.c_int
            L.orc_query_sigma.argtypes = [dp, i, i, i, i, dp]
            L.orc_mean_cov.argtypes = [dp, i, i, i, i, dp, dp]
            L.orc_hadamard.argtypes = [dp, dp, i, i]
            L.orc_jacobi.argtypes = [dp, i, ctypes.c_double, i, dp, dp]
            L.orc_jacobi.restype = ctypes.c_int
            L.orc_select_topr.argtypes = [dp, i, i, up, ip]
            L.orc_select_topr.restype = ctypes.c_int
            L.orc_rotation.argtypes = [dp, ip, i, i, dp, dp, dp]
            L.orc_dmu_from_R.argtypes = [dp, i, i, i, dp, dp]
            L.orc_calibrate.argtypes = [dp, dp, i, i, i, i, i, i, i, i, ctypes.c_double, i,
                                        dp, dp, dp, dp, dp, up, ip, dp, dp, ip]
            L.orc_calibrate.restype = ctypes.c_int
            L.orc_compress.argtypes = [dp, dp, i, i, i, i, dp]
            L.orc_round_bf16.argtypes = [ctypes.c_double]
            L.orc_round_bf16.restype = ctypes.c_double
            L.orc_round_bf16_array.argtypes = [dp, ctypes.c_size_t, dp]
            L.orc_round_f32_array.argtypes = [dp, ctypes.c_size_t, dp]
            L.orc_decode.argtypes = [i, i, i, i, i, i, dp, dp, dp, dp, dp, dp, dp,
                                     ctypes.c_double, dp]
            L.orc_scores.argtypes = [i, i, i, i, i, i, dp, dp, dp, dp, dp, ctypes.c_double, dp]
            L.orc_subspace.argtypes = [dp, dp, i, i, i, ctypes.c_double, dp]
            L.orc_subspace.restype = ctypes.c_int
            L.orc_budget.argtypes = [ctypes.c_double, ctypes.c_double]
            L.orc_budget.restype = ctypes.c_double
            _lib = L
    return _lib


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _p(a: np.ndarray, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


# --------------------------------------------------------------------------
# Alg. 1 step by step
# --------------------------------------------------------------------------
def query_sigma(Qw, W=None) -> np.ndarray:
    """sigma[u, j] = ||Qw[u, :, :, j]||_2 over the G*W window rows.
    Qw: [U, G, W, d].  W == 0 (or Qw None with W=0) -> ones."""
    Qw = _f64(Qw)
    U, G, Wd, d = Qw.shape
    out = np.empty((U, d))
    lib().orc_query_sigma(_p(Qw), U, G, Wd if W is None else W, d, _p(out))
    return out


def mean_cov(K, center=True):
    """mu [U, d] and C [U, d, d] = (K - mu)^T (K - mu), two-pass (Alg. 1 l.1-3)."""
    K = _f64(K)
    U, N, d = K.shape
    mu = np.empty((U, d))
    C = np.empty((U, d, d))
    lib().orc_mean_cov(_p(K), U, N, d, int(bool(center)), _p(mu), _p(C))
    return mu, C


def hadamard(C, sigma) -> np.ndarray:
    """C_q = (sigma sigma^T) (.) C, symmetrised (Alg. 1 l.5)."""
    Cq = _f64(C).copy()
    sigma = _f64(sigma)
    U, d, _ = Cq.shape
    lib().orc_hadamard(_p(Cq), _p(sigma), U, d)
    return Cq


def jacobi(A, tol=JACOBI_TOL, max_sweeps=JACOBI_MAX_SWEEPS):
    """Cyclic Jacobi: returns (lam [d] in solver order, V [d, d], sweeps)."""
    A = _f64(A)
    d = A.shape[0]
    lam = np.empty(d)
    V = np.empty((d, d))
    sw = lib().orc_jacobi(_p(A), d, float(tol), int(max_sweeps), _p(lam), _p(V))
    return lam, V, sw


def select_topr(lam, r):
    """(mask [ceil(d/32)] uint32, idx [r] int32 ascending) or None on NaN."""
    lam = _f64(lam)
    d = lam.shape[0]
    mask = np.zeros((d + 31) // 32, dtype=np.uint32)
    idx = np.zeros(r, dtype=np.int32)
    rc = lib().orc_select_topr(_p(lam), d, int(r), _p(mask, ctypes.c_uint32),
                               _p(idx, ctypes.c_int32))
    return None if rc != 0 else (mask, idx)


def rotation(V, idx, mu):
    """R_r = V[:, idx], delta_mu = mu - R_r R_r^T mu (Alg. 1 l.15)."""
    V = _f64(V)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    mu = _f64(mu)
    d = V.shape[0]
    r = idx.shape[0]
    Rr = np.empty((d, r))
    dmu = np.empty(d)
    lib().orc_rotation(_p(V), _p(idx, ctypes.c_int32), d, r, _p(mu), _p(Rr), _p(dmu))
    return Rr, dmu


def dmu_from_R(Rr, mu):
    """delta_mu = mu - R R^T mu for a given (e.g. stored) R: Rr [U, d, r], mu [U, d]."""
    Rr = _f64(Rr)
    mu = _f64(mu)
    U, d, r = Rr.shape
    out = np.empty((U, d))
    lib().orc_dmu_from_R(_p(Rr), U, d, r, _p(mu), _p(out))
    return out


def calibrate(K, Qw, r, center=True, query_weight=True, tol=JACOBI_TOL,
              max_sweeps=JACOBI_MAX_SWEEPS) -> dict:
    """Alg. 1 steps 1-6 with an exact eigendecomposition.

    K [U, N, d]; Qw [U, G, W, d] (W may be 0) -> dict of fp64 arrays."""
    K = _f64(K)
    U, N, d = K.shape
    if Qw is None:
        Qw = np.zeros((U, 1, 0, d))
    Qw = _f64(Qw)
    _, G, W, _ = Qw.shape
    words = (d + 31) // 32
    out = dict(sigma=np.empty((U, d)), mu=np.empty((U, d)), Cq=np.empty((U, d, d)),
               lam=np.empty((U, d)), V=np.empty((U, d, d)),
               mask=np.zeros((U, words), dtype=np.uint32), idx=np.zeros((U, r), dtype=np.int32),
               R=np.empty((U, d, r)), dmu=np.empty((U, d)), sweeps=np.zeros(U, dtype=np.int32))
    rc = lib().orc_calibrate(
        _p(K), _p(Qw), U, G, N, d, W, int(r), int(bool(center)), int(bool(query_weight)),
        float(tol), int(max_sweeps), _p(out["sigma"]), _p(out["mu"]), _p(out["Cq"]),
        _p(out["lam"]), _p(out["V"]), _p(out["mask"], ctypes.c_uint32),
        _p(out["idx"], ctypes.c_int32), _p(out["R"]), _p(out["dmu"]),
        _p(out["sweeps"], ctypes.c_int32))
    out["ok"] = rc == 0
    return out


def state_doubles(d: int) -> int:
    return d * d + 2 * d + 2


def calib_state(K, Qw, state_units, query_weight=True, state=None) -> np.ndarray:
    """NEXT-3 / calibrate-side token sharding: the sums behind Alg. 1 l.1-5 per
    state entry s, adding every unit u with u % state_units == s (ascending u):
        S = sum_n k_n k_n^T, colsum = sum_n k_n, sigma2_j = sum_window q_j^2, count = #tokens.
    Returns (or adds into) [state_units, d*d + 2d + 2] fp64 (layout of rotatek_calib_accumulate)."""
    K = _f64(K)
    U, N, d = K.shape
    if state is None:
        state = np.zeros((state_units, state_doubles(d)))
    for u in range(U):
        s = u % state_units
        S = state[s, : d * d].reshape(d, d)
        S += K[u].T @ K[u]
        state[s, d * d: d * d + d] += K[u].sum(axis=0)
        if query_weight and Qw is not None and Qw.shape[2] > 0:
            state[s, d * d + d: d * d + 2 * d] += (_f64(Qw[u]) ** 2).sum(axis=(0, 1))
        state[s, d * d + 2 * d] += N
    return state


def calibrate_from_state(state, r, center=True, query_weight=True, tol=JACOBI_TOL,
                         max_sweeps=JACOBI_MAX_SWEEPS) -> dict:
    """Alg. 1 l.1-6 from pooled sums: mu = colsum / count, C = S - count mu mu^T,
    C_q = (sigma sigma^T) (.) C with sigma = sqrt(sigma2) (pooled as Q4) or 1,
    then the exact eigendecomposition, top-r select and delta_mu of calibrate()."""
    state = _f64(state)
    nS = state.shape[0]
    d = int(round((-2 + np.sqrt(4 + 4 * (state.shape[1] - 2))) / 2))
    out = dict(mu=np.empty((nS, d)), Cq=np.empty((nS, d, d)), lam=np.empty((nS, d)),
               R=np.empty((nS, d, r)), dmu=np.empty((nS, d)),
               mask=np.zeros((nS, (d + 31) // 32), dtype=np.uint32), idx=np.zeros((nS, r), np.int32))
    for s in range(nS):
        S = state[s, : d * d].reshape(d, d)
        col = state[s, d * d: d * d + d]
        n = state[s, d * d + 2 * d]
        mu = col / n if center else np.zeros(d)
        C = S - n * np.outer(mu, mu)
        sig = np.sqrt(state[s, d * d + d: d * d + 2 * d]) if query_weight else np.ones(d)
        Cq = np.outer(sig, sig) * C
        Cq = 0.5 * (Cq + Cq.T)
        lam, V, _ = jacobi(Cq, tol, max_sweeps)
        mask, idx = select_topr(lam, r)
        Rr, dmu = rotation(V, idx, mu)
        out["mu"][s], out["Cq"][s], out["lam"][s] = mu, Cq, lam
        out["R"][s], out["dmu"][s], out["mask"][s], out["idx"][s] = Rr, dmu, mask, idx
    return out


def compress(K, R) -> np.ndarray:
    """K~ = K R_r in fp64 (Alg. 1 l.14), before the quantisation point."""
    K = _f64(K)
    R = _f64(R)
    U, N, d = K.shape
    r = R.shape[2]
    Kt = np.empty((U, N, r))
    lib().orc_compress(_p(K), _p(R), U, N, d, r, _p(Kt))
    return Kt


def quantize(x, dtype: str) -> np.ndarray:
    """The quantisation point: RNE of fp64 values to the cache dtype
    ('bf16' or 'f32'), returned as fp64 holding exactly the rounded values."""
    x = _f64(x)
    y = np.empty_like(x)
    if dtype == "bf16":
        lib().orc_round_bf16_array(_p(x), x.size, _p(y))
    elif dtype == "f32":
        lib().orc_round_f32_array(_p(x), x.size, _p(y))
    else:
        raise ValueError(dtype)
    return y


def round_bf16_scalar(x: float) -> float:
    return lib().orc_round_bf16(float(x))


def decode(q, Kt, V, R, dmu, Ktext=None, Vtext=None, scale=0.0) -> np.ndarray:
    """Alg. 2 per unit and query head: q [U, G, d], Kt [U, N, r], V [U, N, d],
    R [U, d, r], dmu [U, d] or None, Ktext/Vtext [U, M, d] or None -> out [U, G, d]."""
    q = _f64(q)
    Kt = _f64(Kt)
    V = _f64(V)
    R = _f64(R)
    U, G, d = q.shape
    N, r = Kt.shape[1], Kt.shape[2]
    if Ktext is None:
        Ktext = np.zeros((U, 0, d))
        Vtext = np.zeros((U, 0, d))
    Ktext = _f64(Ktext)
    Vtext = _f64(Vtext)
    M = Ktext.shape[1]
    out = np.empty((U, G, d))
    dm = None if dmu is None else _f64(dmu)
    lib().orc_decode(U, G, d, r, N, M, _p(q), _p(Kt), _p(V), _p(R),
                     None if dm is None else _p(dm), _p(Ktext), _p(Vtext), float(scale),
                     _p(out))
    return out


def decode_partial(q, Kt, V, R, dmu, Ktext=None, Vtext=None, scale=0.0) -> np.ndarray:
    """Alg. 2 over ONE token shard, stopped before the normalisation: the online-softmax
    state of App. C per unit and query head, written out from its definition:
        z_n = s_n log2(e)  (s_n the scaled scores of Alg. 2 l.3-4, visual then text),
        m = max_n z_n,  l = sum_n 2^(z_n - m),  acc = sum_n 2^(z_n - m) V_n.
    Returns [U, G, d + 2] = acc | m | l (the layout of rotatek_decode_attn_partial)."""
    s = scores(q, Kt, R, dmu, Ktext, scale) * np.log2(np.e)       # [U, G, N + M]
    Vall = _f64(V) if Vtext is None else np.concatenate([_f64(V), _f64(Vtext)], axis=1)
    m = s.max(axis=2)
    w = np.exp2(s - m[:, :, None])
    U, G, _ = s.shape
    out = np.empty((U, G, Vall.shape[2] + 2))
    out[:, :, :-2] = np.einsum("ugn,und->ugd", w, Vall)
    out[:, :, -2] = m
    out[:, :, -1] = w.sum(axis=2)
    return out


def merge_partials(parts) -> np.ndarray:
    """Merge token-shard states [P, U, G, d+2]: M = max_p m_p,
    out = sum_p 2^(m_p - M) acc_p / sum_p 2^(m_p - M) l_p."""
    parts = _f64(parts)
    m = parts[..., -2]
    M = m.max(axis=0)
    f = np.exp2(m - M[None])
    acc = (parts[..., :-2] * f[..., None]).sum(axis=0)
    return acc / (parts[..., -1] * f).sum(axis=0)[..., None]


def scores(q, Kt, R, dmu, Ktext=None, scale=0.0) -> np.ndarray:
    """Alg. 2 lines 1-5: concatenated scores [U, G, N + M] (visual first)."""
    q = _f64(q)
    Kt = _f64(Kt)
    R = _f64(R)
    U, G, d = q.shape
    N, r = Kt.shape[1], Kt.shape[2]
    if Ktext is None:
        Ktext = np.zeros((U, 0, d))
    Ktext = _f64(Ktext)
    M = Ktext.shape[1]
    out = np.empty((U, G, N + M))
    dm = None if dmu is None else _f64(dmu)
    lib().orc_scores(U, G, d, r, N, M, _p(q), _p(Kt), _p(R), None if dm is None else _p(dm),
                     _p(Ktext), float(scale), _p(out))
    return out


SUBSPACE_T = 5          # "T = 5 iterations"
SUBSPACE_EPS = 1e-6     # ridge factor: unspecified in the paper; SPEC's default


def subspace(Cq, V0, T=SUBSPACE_T, eps=SUBSPACE_EPS):
    """NEXT-1, Alg. 1 lines 6-13: Cholesky-QR subspace iteration from the given V0.
    Cq [U, d, d] (or [d, d]), V0 [U, d, k] (or [d, k]) -> R_k of the same shape as V0.
    Returns None if a Cholesky pivot fails."""
    Cq = _f64(Cq)
    V0 = _f64(V0)
    single = Cq.ndim == 2
    if single:
        Cq, V0 = Cq[None], V0[None]
    U, d, k = V0.shape
    out = np.empty((U, d, k))
    for u in range(U):
        c = np.ascontiguousarray(Cq[u])
        v = np.ascontiguousarray(V0[u])
        o = np.empty((d, k))
        if lib().orc_subspace(_p(c), _p(v), d, k, int(T), float(eps), _p(o)) != 0:
            return None
        out[u] = o
    return out[0] if single else out


def calibrate_subspace(K, Qw, V0, T=SUBSPACE_T, eps=SUBSPACE_EPS, center=True,
                       query_weight=True) -> dict:
    """Alg. 1 with the paper's default solver: steps 1-5 as in calibrate(), the basis from
    subspace(), then delta_mu = mu - R R^T mu (line 15)."""
    K = _f64(K)
    U, N, d = K.shape
    if Qw is None or not query_weight:
        Qw = np.zeros((U, 1, 0, d))
    sig = query_sigma(Qw)
    mu, C = mean_cov(K, center)
    Cq = hadamard(C, sig)
    R = subspace(Cq, V0, T, eps)
    return dict(sigma=sig, mu=mu, Cq=Cq, R=R, dmu=dmu_from_R(R, mu) if center else np.zeros((U, d)))


def budget(token_keep: float, channel_keep: float) -> float:
    """Visual KV-cache multiplier token_keep * (1 + channel_keep) / 2 (tab:main_comparison)."""
    return lib().orc_budget(float(token_keep), float(channel_keep))


def pipeline(K, V, Qw, q, r, dtype="bf16", Ktext=None, Vtext=None, center=True,
             query_weight=True, scale=0.0) -> dict:
    """Oracle steps 1-8 end to end with the quantisation point of step 7:
    K~ = RNE_dtype(K R_r) (R_r, delta_mu kept in fp64)."""
    cal = calibrate(K, Qw, r, center=center, query_weight=query_weight)
    Kt = quantize(compress(K, cal["R"]), dtype)
    out = decode(q, Kt, V, cal["R"], cal["dmu"] if center else None, Ktext, Vtext, scale)
    cal["Kt"] = Kt
    cal["out"] = out
    return cal
