"""The C-ABI library: it loads, exports every symbol include/rotatek.h declares, and its
host-side validation returns the documented status codes (no GPU needed: every call here
fails validation before any CUDA work is enqueued)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rotatek.h")
LIB = os.path.join(ROOT, "paper_2605_19218_b200", "librotatek.so")


@pytest.fixture(scope="module")
def rk():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-j8", "-C", ROOT, "paper_2605_19218_b200/librotatek.so"])
    from paper_2605_19218_b200 import rotatek
    return rotatek


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rotatek_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_three_paper_calls():
    names = _declared_functions()
    for n in ("rotatek_calibrate", "rotatek_compress_kv", "rotatek_decode_attn"):
        assert n in names


def test_exports_every_declared_symbol(rk):
    L = rk.lib()
    out = subprocess.check_output(["nm", "-D", "--defined-only", LIB]).decode()
    exported = set(re.findall(r" T (rotatek_\w+)", out))
    for name in _declared_functions():
        assert name in exported, name
        assert hasattr(L, name)


def test_version_and_strings(rk):
    L = rk.lib()
    assert L.rotatek_abi_version() == 3  # 2: rotatek_dims.text_stride; 3: token-list prefill, decode kernel 5
    for code in range(7):
        assert L.rotatek_status_string(code).decode().startswith("ROTATEK_")


def test_workspace_bytes(rk):
    d = rk.make_dims(1024, 1, 128, 32, 2880, 128, 32, rk.BF16)
    assert rk.workspace_bytes(d, rk.OP_CALIBRATE) > 1024 * 128 * 128 * 8
    assert rk.workspace_bytes(d, rk.OP_DECODE) >= 1024 * 4
    bad = rk.make_dims(0, 1, 128, 32, 2880, 128, 32, rk.BF16)
    assert rk.workspace_bytes(bad, rk.OP_DECODE) == 0


def _calib(rk, dims, K=0x1000, Qw=0x2000, R=0x3000, dmu=0x4000, ws=0x5000, nws=1 << 40):
    L = rk.lib()
    vp = ctypes.c_void_p
    return L.rotatek_calibrate(ctypes.byref(dims), rk.DEFAULT_FLAGS, vp(K), vp(Qw), vp(R), vp(dmu),
                               None, None, None, None, None, vp(ws), nws, None)


@pytest.mark.parametrize("field,value", [("units", 0), ("group", 0), ("head_dim", 24),
                                         ("head_dim", 512), ("rank", 0), ("rank", 129),
                                         ("n_vis", 0), ("n_text", -1), ("q_window", -2)])
def test_calibrate_dims_errors(rk, field, value):
    d = rk.make_dims(4, 1, 128, 32, 100, 0, 32, rk.BF16)
    setattr(d, field, value)
    assert _calib(rk, d) == rk.ERR_DIMS


def test_calibrate_null_align_workspace_unsupported(rk):
    d = rk.make_dims(4, 1, 128, 32, 100, 0, 32, rk.BF16)
    assert _calib(rk, d, K=0) == rk.ERR_NULL
    assert _calib(rk, d, Qw=0) == rk.ERR_DIMS            # W > 0 needs Qw
    assert _calib(rk, d, R=0x3004) == rk.ERR_ALIGN
    assert _calib(rk, d, nws=16) == rk.ERR_WORKSPACE
    assert "workspace" in rk.lib().rotatek_last_error().decode()
    d256 = rk.make_dims(4, 1, 256, 32, 100, 0, 32, rk.BF16)
    assert _calib(rk, d256) == rk.ERR_UNSUPPORTED


def test_decode_errors(rk):
    L = rk.lib()
    vp = ctypes.c_void_p
    d = rk.make_dims(4, 7, 128, 32, 100, 16, 0, rk.BF16)

    def call(ktext=0x6000, ws=0x7000, nws=1 << 40, q=0x1000, kernel=0):
        return L.rotatek_decode_attn_ex(ctypes.byref(d), vp(q), vp(0x2000), vp(0x3000),
                                        vp(0x4000), vp(0x5000), vp(ktext), vp(0x6100), 0.0,
                                        vp(0x8000), vp(ws), nws, 0, kernel, None)
    assert call(q=0) == rk.ERR_NULL
    assert call(ktext=0) == rk.ERR_NULL                  # M > 0 needs the text segment
    assert call(nws=8) == rk.ERR_WORKSPACE
    assert call(q=0x1008) == rk.ERR_ALIGN
    assert call(kernel=6) == rk.ERR_DIMS


def test_decode_varlen_errors(rk):
    """rotatek_decode_attn_varlen: host validation of the length arrays and the shared
    rotation (no compute call: nothing here reaches a kernel launch)."""
    L = rk.lib()
    vp = ctypes.c_void_p
    d = rk.make_dims(4, 7, 128, 32, 100, 16, 0, rk.BF16)

    def call(nv=0x9000, nt=0x9100, r_units=0, q=0x1000, nws=8):
        return L.rotatek_decode_attn_varlen(ctypes.byref(d), r_units, vp(nv), vp(nt), vp(q),
                                            vp(0x2000), vp(0x3000), vp(0x4000), vp(0x5000),
                                            vp(0x6000), vp(0x6100), 0.0, vp(0x8000), vp(0x7000),
                                            nws, 0, 0, None)
    assert call(nv=0x9004) == rk.ERR_ALIGN
    assert call(nt=0x9104) == rk.ERR_ALIGN
    assert call(q=0) == rk.ERR_NULL
    assert call(nws=8) == rk.ERR_WORKSPACE
    assert call(nws=1 << 40, r_units=3) == rk.ERR_DIMS    # r_units must divide units


def test_compress_and_select_errors(rk):
    L = rk.lib()
    vp = ctypes.c_void_p
    d = rk.make_dims(4, 1, 128, 32, 100, 0, 0, rk.BF16)
    assert L.rotatek_compress_kv(ctypes.byref(d), vp(0), vp(0x2000), vp(0x3000), None) == rk.ERR_NULL
    assert L.rotatek_select_topr(4, 128, 0, vp(0x1000), vp(0x2000), vp(0x3000), None, None) == rk.ERR_DIMS
    assert L.rotatek_select_topr(4, 128, 8, vp(0x1004), vp(0x2000), vp(0x3000), None, None) == rk.ERR_ALIGN


def test_binding_rejects_missing_library(tmp_path, monkeypatch):
    """The product path fails loudly when the CUDA library is absent (no fallback)."""
    from paper_2605_19218_b200 import rotatek
    monkeypatch.setattr(rotatek, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(rotatek, "_lib", None)
    with pytest.raises(RuntimeError, match="missing"):
        rotatek.lib()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_19218_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src, f
                assert "liboracle" not in src and "orc_" not in src, f


def test_token_prefill_host_validation(rk):
    """rotatek_calibrate_tokens / rotatek_compress_kv_tokens: misaligned token arrays, a token
    list without n_src, and shapes without the tensor-core path fail before any CUDA work."""
    L = rk.lib()
    vp = ctypes.c_void_p
    d = rk.make_dims(4, 1, 128, 32, 300, 0, 32, rk.BF16)

    def cal(dims, n_src=500, idx=0x7000, nvu=None):
        return L.rotatek_calibrate_tokens(ctypes.byref(dims), rk.DEFAULT_FLAGS, vp(0x1000), n_src, vp(idx),
                                          vp(nvu), vp(0x2000), vp(0x3000), vp(0x4000), None, None, None,
                                          None, None, vp(0x5000), 1 << 40, None)

    def cmp(dims, n_src=500, idx=0x7000, nvu=None):
        return L.rotatek_compress_kv_tokens(ctypes.byref(dims), 0, vp(0x1000), n_src, vp(idx), vp(nvu),
                                            vp(0x3000), vp(0x6000), None)

    assert cal(d, idx=0x7004) == rk.ERR_ALIGN
    assert cal(d, idx=None, nvu=0x7008) == rk.ERR_ALIGN
    assert cal(d, n_src=0) == rk.ERR_DIMS
    assert cmp(d, idx=0x7004) == rk.ERR_ALIGN
    assert cmp(d, n_src=0) == rk.ERR_DIMS
    f32 = rk.make_dims(4, 1, 128, 32, 300, 0, 32, rk.F32)      # no tensor-core path
    assert cal(f32) == rk.ERR_UNSUPPORTED
    assert cmp(f32) == rk.ERR_UNSUPPORTED
    d64 = rk.make_dims(4, 1, 64, 16, 300, 0, 32, rk.BF16)      # d != 128
    assert cal(d64) == rk.ERR_UNSUPPORTED
    assert cmp(d64) == rk.ERR_UNSUPPORTED


def test_flag_values_match_header(rk):
    """The binding's flag constants are the header's enum values (a mismatch would silently
    select another solver or drop the centering)."""
    src = open(HEADER).read()
    flags = {m.group(1): 1 << int(m.group(2))
             for m in re.finditer(r"ROTATEK_([A-Z0-9_]+)\s*=\s*1u\s*<<\s*(\d+)\s*,", src)}
    for name in ("CENTER", "QUERY_WEIGHT", "EIG_FP64", "EIG_TWOSIDED", "SIMT_ONLY"):
        assert getattr(rk, name) == flags[name], name
    assert rk.DEFAULT_FLAGS == flags["CENTER"] | flags["QUERY_WEIGHT"]
