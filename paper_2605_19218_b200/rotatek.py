"""Thin Python binding of librotatek.so (include/rotatek.h).

Argument marshalling only: shapes are read from the torch tensors, outputs and
zero-filled workspaces are allocated with torch (device memory is plumbing),
and every step of the hot path runs in the library's sm_100a kernels.  There
is no CPU or PyTorch fallback: if the library is missing or a call fails, a
RuntimeError is raised.

Names follow the paper: K (visual keys), Qw (query window Q_W), R (R_r, the kept
eigenvectors), dmu (delta_mu), K_comp (K~), K_text/V_text (prompt+text K_pt, V).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ROTATEK_LIB") or os.path.join(_HERE, "librotatek.so")  # A/B builds

OK, ERR_NULL, ERR_DIMS, ERR_ALIGN, ERR_WORKSPACE, ERR_UNSUPPORTED, ERR_CUDA = range(7)
BF16, F32 = 0, 1
CENTER, QUERY_WEIGHT, EIG_FP64, EIG_TWOSIDED, SIMT_ONLY = 1, 2, 4, 8, 256
DEFAULT_FLAGS = CENTER | QUERY_WEIGHT
OP_CALIBRATE, OP_DECODE = 0, 1
KERNEL_AUTO, KERNEL_GENERIC, KERNEL_FAST, KERNEL_GQA, KERNEL_STEAL, KERNEL_GQA_WARP = 0, 1, 2, 3, 4, 5
DECODE_OVERLAP = 0x100  # OR into kernel: programmatic dependent launch (include/rotatek.h)


class Dims(ctypes.Structure):
    _fields_ = [("units", ctypes.c_int32), ("group", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("n_vis", ctypes.c_int32), ("n_text", ctypes.c_int32),
                ("q_window", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("text_stride", ctypes.c_int32)]


class RotateKError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(what)


_lock = threading.Lock()
_lib = None


def lib():
    """Load librotatek.so (fails loudly if it has not been built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or "
                                   "`python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            vp, sz, u32, i32, f = (ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32,
                                   ctypes.c_int32, ctypes.c_float)
            dp = ctypes.POINTER(Dims)
            L.rotatek_workspace_bytes.argtypes = [dp, ctypes.c_int]
            L.rotatek_workspace_bytes.restype = sz
            L.rotatek_calibrate.argtypes = [dp, u32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
            L.rotatek_calibrate_subspace.argtypes = [dp, u32, vp, vp, vp, i32, f, vp, vp, vp, vp,
                                                     vp, sz, vp]
            L.rotatek_calibrate_subspace.restype = ctypes.c_int
            L.rotatek_compress_kv.argtypes = [dp, vp, vp, vp, vp]
            L.rotatek_compress_kv_ex.argtypes = [dp, vp, vp, vp, u32, vp]
            L.rotatek_decode_attn.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, f, vp, vp, sz, vp]
            L.rotatek_decode_attn_ex.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, f, vp, vp, sz,
                                                 i32, i32, vp]
            L.rotatek_select_topr.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp]
            L.rotatek_decode_attn_partial.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, f, vp, vp, sz, vp]
            L.rotatek_decode_attn_ex2.argtypes = [dp, i32, vp, vp, vp, vp, vp, vp, vp, f, vp, vp, sz,
                                                  i32, i32, vp]
            L.rotatek_decode_attn_varlen.argtypes = [dp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                     f, vp, vp, sz, i32, i32, vp]
            L.rotatek_compress_kv_ex2.argtypes = [dp, i32, vp, vp, vp, u32, vp]
            L.rotatek_calib_accumulate.argtypes = [dp, u32, vp, vp, i32, vp, vp, sz, vp]
            L.rotatek_calibrate_from_state.argtypes = [dp, u32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                       sz, vp]
            L.rotatek_merge_partials.argtypes = [i32, i32, i32, i32, vp, vp, vp]
            L.rotatek_calibrate_tokens.argtypes = [dp, u32, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                                   vp, vp, sz, vp]
            L.rotatek_compress_kv_tokens.argtypes = [dp, i32, vp, i32, vp, vp, vp, vp, vp]
            L.rotatek_gather_tokens.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp]
            for fn in ("rotatek_calibrate", "rotatek_compress_kv", "rotatek_compress_kv_ex",
                       "rotatek_decode_attn",
                       "rotatek_decode_attn_ex", "rotatek_select_topr", "rotatek_decode_attn_partial",
                       "rotatek_merge_partials", "rotatek_decode_attn_ex2", "rotatek_compress_kv_ex2",
                       "rotatek_calib_accumulate", "rotatek_calibrate_from_state",
                       "rotatek_gather_tokens", "rotatek_decode_attn_varlen",
                       "rotatek_calibrate_tokens", "rotatek_compress_kv_tokens"):
                getattr(L, fn).restype = ctypes.c_int
            L.rotatek_status_string.argtypes = [ctypes.c_int]
            L.rotatek_status_string.restype = ctypes.c_char_p
            L.rotatek_last_error.restype = ctypes.c_char_p
            L.rotatek_abi_version.restype = ctypes.c_int
            L.rotatek_last_launch_count.restype = ctypes.c_int
            L.rotatek_debug_decode_trace.argtypes = [vp]
            L.rotatek_debug_decode_trace.restype = None
            _lib = L
    return _lib


def _check(status: int):
    if status != OK:
        L = lib()
        raise RotateKError(status, f"{L.rotatek_status_string(status).decode()}: "
                                   f"{L.rotatek_last_error().decode()}")


def last_launch_count() -> int:
    return lib().rotatek_last_launch_count()


def debug_decode_trace(buf: torch.Tensor | None):
    """Diagnostics: per-warp globaltimer stamps of the streaming decode kernels into
    buf (int64 device tensor of >= 8 * warps), or None to uninstall."""
    lib().rotatek_debug_decode_trace(None if buf is None else ctypes.c_void_p(buf.data_ptr()))


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}; use bfloat16 or float32")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("librotatek takes device tensors")
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _check_decode_dtypes(q, K_comp, V, R, dmu, K_text, V_text):
    """The ABI reads q, V and the text K/V as K_comp's dtype and R, dmu as fp32: reject a
    mismatch here instead of letting the kernel reinterpret the bytes."""
    dt = K_comp.dtype
    for name, t in (("q", q), ("V", V), ("K_text", K_text), ("V_text", V_text)):
        if t is not None and t.dtype != dt:
            raise TypeError(f"{name} is {t.dtype} but K_comp is {dt}: all cache tensors and q "
                            "must share one dtype")
    for name, t in (("R", R), ("dmu", dmu)):
        if t is not None and t.dtype != torch.float32:
            raise TypeError(f"{name} must be float32 (got {t.dtype})")


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def make_dims(units, group, head_dim, rank, n_vis, n_text=0, q_window=0, dtype=BF16,
              text_stride=0) -> Dims:
    return Dims(int(units), int(group), int(head_dim), int(rank), int(n_vis), int(n_text),
                int(q_window), int(dtype), int(text_stride))


def workspace_bytes(dims: Dims, op: int) -> int:
    return int(lib().rotatek_workspace_bytes(ctypes.byref(dims), op))


_ws_cache: dict = {}


def workspace(dims: Dims, op: int, device, stream=None) -> torch.Tensor:
    """Zero-filled workspace for calls enqueued on `stream` (default: the current stream).

    The ABI requires zeros on first use and every call leaves the counter region zeroed
    (include/rotatek.h), so one buffer is kept per (device, op, stream, units) -- calls on
    different streams never share counters -- and replaced by a larger zero-filled one
    (allocated and zeroed ON that stream) when a shape needs more, e.g. an appendable text
    segment growing during generation.  The decode counter region's offsets depend on the
    unit count only, so a larger buffer serves every smaller shape of the same units."""
    n = workspace_bytes(dims, op)
    if n == 0:
        _check(ERR_DIMS)
    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    s = torch.cuda.current_stream(dev) if stream is None else stream
    key = (str(dev), op, s.cuda_stream, int(dims.units) if op == OP_DECODE else 0)
    t = _ws_cache.get(key)
    if t is None or t.numel() < n:
        with torch.cuda.stream(s):
            t = torch.zeros(max(n, 0 if t is None else t.numel()), dtype=torch.uint8, device=dev)
        _ws_cache[key] = t
    return t


# --------------------------------------------------------------------------- calibrate
def _tok_args(K, tok_idx, n_vis_u, n_log):
    """Checks of the token-selection inputs (include/rotatek.h, rotatek_calibrate_tokens)."""
    U = K.shape[0]
    if tok_idx is not None:
        assert tok_idx.dtype == torch.int32 and tok_idx.shape == (U, n_log) and tok_idx.is_cuda
    if n_vis_u is not None:
        assert n_vis_u.dtype == torch.int32 and n_vis_u.shape == (U,) and n_vis_u.is_cuda


def calibrate(K: torch.Tensor, Qw: torch.Tensor | None, rank: int, flags: int = DEFAULT_FLAGS,
              *, want_full: bool = False, tok_idx: torch.Tensor | None = None,
              n_vis_u: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> dict:
    """Alg. 1 steps 1-5 (+ select, delta_mu).  K [U, N, d]; Qw [U, G, W, d] or None.
    tok_idx [U, n] int32: calibrate on rows tok_idx[u] of K [U, n_src, d] (token pruning
    survivors, gathered by the kernel); n_vis_u [U] int32: per-unit valid token counts
    (rotatek_calibrate_tokens).  flags: CENTER | QUERY_WEIGHT (default), EIG_FP64 (fp64
    Jacobi), EIG_TWOSIDED (two-sided instead of the default one-sided fp32 Jacobi, d = 128),
    SIMT_ONLY (CUDA-core covariance) -- include/rotatek.h.

    Returns dict(R [U,d,r] f32, dmu [U,d] f32, eigvals [U,d] f32, mask [U,ceil(d/32)] i32
    (uint32 bit pattern), idx [U,r] i32, info [U] i32, R_full [U,d,d] f32 if want_full)."""
    U, N, d = K.shape
    n_src = N
    if tok_idx is not None:
        N = tok_idx.shape[1]
    _tok_args(K, tok_idx, n_vis_u, N)
    if Qw is None:
        G, W = 1, 0
    else:
        assert Qw.dim() == 4 and Qw.shape[0] == U and Qw.shape[3] == d and Qw.dtype == K.dtype
        G, W = Qw.shape[1], Qw.shape[2]
    dims = make_dims(U, G, d, rank, N, 0, W, _dtype_code(K))
    dev = K.device
    out = dict(
        R=torch.empty((U, d, rank), dtype=torch.float32, device=dev),
        dmu=torch.empty((U, d), dtype=torch.float32, device=dev),
        eigvals=torch.empty((U, d), dtype=torch.float32, device=dev),
        mask=torch.empty((U, (d + 31) // 32), dtype=torch.int32, device=dev),
        idx=torch.empty((U, rank), dtype=torch.int32, device=dev),
        info=torch.empty((U,), dtype=torch.int32, device=dev),
    )
    out["R_full"] = torch.empty((U, d, d), dtype=torch.float32, device=dev) if want_full else None
    if ws is None:
        ws = workspace(dims, OP_CALIBRATE, dev, stream)
    if tok_idx is None and n_vis_u is None:
        _check(lib().rotatek_calibrate(ctypes.byref(dims), flags, _ptr(K),
                                       _ptr(Qw) if W > 0 else None, _ptr(out["R"]), _ptr(out["dmu"]),
                                       _ptr(out["eigvals"]), _ptr(out["mask"]), _ptr(out["idx"]),
                                       _ptr(out["R_full"]), _ptr(out["info"]), _ptr(ws), ws.numel(),
                                       _stream(stream)))
    else:
        _check(lib().rotatek_calibrate_tokens(ctypes.byref(dims), flags, _ptr(K), n_src, _ptr(tok_idx),
                                              _ptr(n_vis_u), _ptr(Qw) if W > 0 else None, _ptr(out["R"]),
                                              _ptr(out["dmu"]), _ptr(out["eigvals"]), _ptr(out["mask"]),
                                              _ptr(out["idx"]), _ptr(out["R_full"]), _ptr(out["info"]),
                                              _ptr(ws), ws.numel(), _stream(stream)))
    return out


def calibrate_subspace(K: torch.Tensor, Qw: torch.Tensor | None, V0: torch.Tensor,
                       flags: int = DEFAULT_FLAGS, iters: int = 5, ridge: float = 1e-6, *,
                       ws: torch.Tensor | None = None, stream=None) -> dict:
    """Alg. 1 with the paper's default solver (Cholesky-QR subspace iteration from V0).
    K [U, N, d]; Qw [U, G, W, d] or None; V0 [U, d, r] f32 -> dict(R, dmu, ritz, info)."""
    U, N, d = K.shape
    r = V0.shape[2]
    assert V0.shape == (U, d, r) and V0.dtype == torch.float32
    if Qw is None:
        G, W = 1, 0
    else:
        G, W = Qw.shape[1], Qw.shape[2]
    dims = make_dims(U, G, d, r, N, 0, W, _dtype_code(K))
    dev = K.device
    out = dict(R=torch.empty((U, d, r), dtype=torch.float32, device=dev),
               dmu=torch.empty((U, d), dtype=torch.float32, device=dev),
               ritz=torch.empty((U, r), dtype=torch.float32, device=dev),
               info=torch.empty((U,), dtype=torch.int32, device=dev))
    if ws is None:
        ws = workspace(dims, OP_CALIBRATE, dev, stream)
    _check(lib().rotatek_calibrate_subspace(
        ctypes.byref(dims), flags, _ptr(K), _ptr(Qw) if W > 0 else None, _ptr(V0), int(iters),
        float(ridge), _ptr(out["R"]), _ptr(out["dmu"]), _ptr(out["ritz"]), _ptr(out["info"]),
        _ptr(ws), ws.numel(), _stream(stream)))
    return out


def state_doubles(d: int) -> int:
    """Doubles per calibration-state entry (ROTATEK_STATE_DOUBLES)."""
    return d * d + 2 * d + 2


def calib_state(state_units: int, head_dim: int, device="cuda") -> torch.Tensor:
    """A zeroed calibration-statistics state [state_units, ROTATEK_STATE_DOUBLES(d)] f64."""
    return torch.zeros((state_units, state_doubles(head_dim)), dtype=torch.float64, device=device)


def calib_accumulate(K: torch.Tensor, Qw: torch.Tensor | None, state: torch.Tensor,
                     flags: int = DEFAULT_FLAGS, *, ws: torch.Tensor | None = None,
                     stream=None) -> torch.Tensor:
    """Add the Alg. 1 sums of K [U, N, d] (and Qw [U, G, W, d]) into state[u % state_units]
    (NEXT-3 offline calibration; token-sharded calibration before an all-reduce)."""
    U, N, d = K.shape
    if Qw is None:
        G, W = 1, 0
    else:
        G, W = Qw.shape[1], Qw.shape[2]
    nS = state.shape[0]
    assert state.shape == (nS, state_doubles(d)) and state.dtype == torch.float64
    dims = make_dims(U, G, d, 1, N, 0, W, _dtype_code(K))
    if ws is None:
        ws = workspace(dims, OP_CALIBRATE, K.device, stream)
    _check(lib().rotatek_calib_accumulate(ctypes.byref(dims), flags, _ptr(K),
                                          _ptr(Qw) if W > 0 else None, nS, _ptr(state), _ptr(ws),
                                          ws.numel(), _stream(stream)))
    return state


def calibrate_from_state(state: torch.Tensor, rank: int, flags: int = DEFAULT_FLAGS,
                         dtype=torch.bfloat16, *, want_full: bool = False,
                         ws: torch.Tensor | None = None, stream=None) -> dict:
    """Alg. 1 from an accumulated state -> dict like calibrate() ([state_units, ...]).
    dtype: the cache dtype the rotation is for (bf16: fp32 Jacobi + fp64 refinement)."""
    nS = state.shape[0]
    d = int(round((-2 + (4 + 4 * (state.shape[1] - 2)) ** 0.5) / 2))
    dims = make_dims(nS, 1, d, rank, 1, 0, 0, BF16 if dtype == torch.bfloat16 else F32)
    dev = state.device
    out = dict(
        R=torch.empty((nS, d, rank), dtype=torch.float32, device=dev),
        dmu=torch.empty((nS, d), dtype=torch.float32, device=dev),
        eigvals=torch.empty((nS, d), dtype=torch.float32, device=dev),
        mask=torch.empty((nS, (d + 31) // 32), dtype=torch.int32, device=dev),
        idx=torch.empty((nS, rank), dtype=torch.int32, device=dev),
        info=torch.empty((nS,), dtype=torch.int32, device=dev),
    )
    out["R_full"] = torch.empty((nS, d, d), dtype=torch.float32, device=dev) if want_full else None
    if ws is None:
        ws = workspace(dims, OP_CALIBRATE, dev, stream)
    _check(lib().rotatek_calibrate_from_state(
        ctypes.byref(dims), flags, _ptr(state), _ptr(out["R"]), _ptr(out["dmu"]),
        _ptr(out["eigvals"]), _ptr(out["mask"]), _ptr(out["idx"]), _ptr(out["R_full"]),
        _ptr(out["info"]), _ptr(ws), ws.numel(), _stream(stream)))
    return out


# --------------------------------------------------------------------------- compress
def compress_kv(K: torch.Tensor, R: torch.Tensor, out: torch.Tensor | None = None,
                stream=None, flags: int = 0, *, tok_idx: torch.Tensor | None = None,
                n_vis_u: torch.Tensor | None = None) -> torch.Tensor:
    """Alg. 1 line 14: K~ = RNE(K R_r).  K [U, N, d], R [U, d, r] f32 -> [U, N, r] K.dtype.
    flags: SIMT_ONLY selects the CUDA-core kernel instead of tcgen05.
    tok_idx [U, n] int32 / n_vis_u [U] int32: token selection as calibrate() (output
    [U, n, r], rows past a unit's count exactly 0; rotatek_compress_kv_tokens)."""
    U, N, d = K.shape
    if tok_idx is not None or n_vis_u is not None:
        n_src = N
        if tok_idx is not None:
            N = tok_idx.shape[1]
        _tok_args(K, tok_idx, n_vis_u, N)
        r = R.shape[2]
        nR = R.shape[0]
        assert R.shape == (nR, d, r) and U % nR == 0 and R.dtype == torch.float32
        if out is None:
            out = torch.empty((U, N, r), dtype=K.dtype, device=K.device)
        dims = make_dims(U, 1, d, r, N, 0, 0, _dtype_code(K))
        _check(lib().rotatek_compress_kv_tokens(ctypes.byref(dims), nR if nR != U else 0, _ptr(K), n_src,
                                                _ptr(tok_idx), _ptr(n_vis_u), _ptr(R), _ptr(out),
                                                _stream(stream)))
        return out
    r = R.shape[2]
    nR = R.shape[0]   # nR < U: shared (offline) rotation, unit u uses R[u % nR]
    assert R.shape == (nR, d, r) and U % nR == 0 and R.dtype == torch.float32
    if out is None:
        out = torch.empty((U, N, r), dtype=K.dtype, device=K.device)
    dims = make_dims(U, 1, d, r, N, 0, 0, _dtype_code(K))
    _check(lib().rotatek_compress_kv_ex2(ctypes.byref(dims), nR if nR != U else 0, _ptr(K), _ptr(R),
                                         _ptr(out), int(flags), _stream(stream)))
    return out


# --------------------------------------------------------------------------- decode
def decode_attn(q: torch.Tensor, K_comp: torch.Tensor, V: torch.Tensor, R: torch.Tensor,
                dmu: torch.Tensor | None, K_text: torch.Tensor | None = None,
                V_text: torch.Tensor | None = None, scale: float = 0.0,
                out: torch.Tensor | None = None, *, splits: int = 0, kernel: int = KERNEL_AUTO,
                n_text: int | None = None, n_vis_u: torch.Tensor | None = None,
                n_text_u: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """Alg. 2 for all query heads: q [U, G, d], K_comp [U, N, r], V [U, N, d], R [U, d, r],
    dmu [U, d] | None, K_text/V_text [U, M_cap, d] | None -> out [U, G, d] f32.
    n_text: the M <= M_cap valid full-d tokens (default M_cap): an appendable segment.
    n_vis_u / n_text_u: int32 [U] device, per-unit valid lengths over padded caches
    (rotatek_decode_attn_varlen)."""
    U, G, d = q.shape
    N, r = K_comp.shape[1], K_comp.shape[2]
    Mcap = 0 if K_text is None else K_text.shape[1]
    M = Mcap if n_text is None else int(n_text)
    nR = R.shape[0]   # nR < U: shared (offline) rotation, unit u uses R[u % nR], dmu[u % nR]
    assert V.shape == (U, N, d) and R.shape == (nR, d, r) and U % nR == 0
    _check_decode_dtypes(q, K_comp, V, R, dmu, K_text, V_text)
    dims = make_dims(U, G, d, r, N, M, 0, _dtype_code(K_comp), Mcap if M else 0)
    if out is None:
        out = torch.empty((U, G, d), dtype=torch.float32, device=q.device)
    if ws is None:
        ws = workspace(dims, OP_DECODE, q.device, stream)
    for lens in (n_vis_u, n_text_u):
        assert lens is None or (lens.dtype == torch.int32 and lens.shape == (U,) and lens.is_cuda)
    _check(lib().rotatek_decode_attn_varlen(ctypes.byref(dims), nR if nR != U else 0,
                                         _ptr(n_vis_u), _ptr(n_text_u), _ptr(q),
                                         _ptr(K_comp), _ptr(V), _ptr(R), _ptr(dmu),
                                         _ptr(K_text) if M else None, _ptr(V_text) if M else None,
                                         float(scale), _ptr(out), _ptr(ws), ws.numel(), int(splits),
                                         int(kernel), _stream(stream)))
    return out


def decode_attn_partial(q: torch.Tensor, K_comp: torch.Tensor, V: torch.Tensor, R: torch.Tensor,
                        dmu: torch.Tensor | None, K_text: torch.Tensor | None = None,
                        V_text: torch.Tensor | None = None, scale: float = 0.0,
                        part: torch.Tensor | None = None, *, ws: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """Alg. 2 over this rank's token shard -> un-normalised state part [U, G, d+2] f32
    (acc[d] | m | l, base-2 logits; include/rotatek.h)."""
    U, G, d = q.shape
    N, r = K_comp.shape[1], K_comp.shape[2]
    M = 0 if K_text is None else K_text.shape[1]
    assert V.shape == (U, N, d) and R.shape == (U, d, r)
    _check_decode_dtypes(q, K_comp, V, R, dmu, K_text, V_text)
    dims = make_dims(U, G, d, r, N, M, 0, _dtype_code(K_comp))
    if part is None:
        part = torch.empty((U, G, d + 2), dtype=torch.float32, device=q.device)
    if ws is None:
        ws = workspace(dims, OP_DECODE, q.device, stream)
    _check(lib().rotatek_decode_attn_partial(ctypes.byref(dims), _ptr(q), _ptr(K_comp), _ptr(V),
                                             _ptr(R), _ptr(dmu), _ptr(K_text) if M else None,
                                             _ptr(V_text) if M else None, float(scale), _ptr(part),
                                             _ptr(ws), ws.numel(), _stream(stream)))
    return part


def merge_partials(parts: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """parts [P, U, G, d+2] f32 (token shards, shard-major) -> out [U, G, d] f32."""
    P, U, G, d2 = parts.shape
    d = d2 - 2
    if out is None:
        out = torch.empty((U, G, d), dtype=torch.float32, device=parts.device)
    _check(lib().rotatek_merge_partials(U, G, d, P, _ptr(parts), _ptr(out), _stream(stream)))
    return out


def gather_tokens(x: torch.Tensor, keep_idx: torch.Tensor, out: torch.Tensor | None = None,
                  err: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Token pruning (NEXT-2): x [U, n_src, ...] -> [U, n_keep, ...] rows keep_idx [U, n_keep]."""
    U, n_src = x.shape[0], x.shape[1]
    n_keep = keep_idx.shape[1]
    assert keep_idx.shape == (U, n_keep) and keep_idx.dtype == torch.int32
    row_bytes = x[0, 0].numel() * x.element_size()
    if out is None:
        out = torch.empty((U, n_keep) + tuple(x.shape[2:]), dtype=x.dtype, device=x.device)
    _check(lib().rotatek_gather_tokens(U, n_src, n_keep, row_bytes, _ptr(keep_idx), _ptr(x),
                                       _ptr(out), _ptr(err), _stream(stream)))
    return out


def select_topr(eigvals: torch.Tensor, rank: int, stream=None):
    """Top-r select on given eigenvalues [U, d] f32 -> (mask [U, ceil(d/32)], idx [U, r], info [U])."""
    U, d = eigvals.shape
    mask = torch.empty((U, (d + 31) // 32), dtype=torch.int32, device=eigvals.device)
    idx = torch.empty((U, rank), dtype=torch.int32, device=eigvals.device)
    info = torch.empty((U,), dtype=torch.int32, device=eigvals.device)
    _check(lib().rotatek_select_topr(U, d, rank, _ptr(eigvals), _ptr(mask), _ptr(idx), _ptr(info),
                                     _stream(stream)))
    return mask, idx, info
