"""B200-native (sm_100a) hot path of RotateK (arxiv 2605.19218).

librotatek.so implements Alg. 1 (calibrate + compress) and Alg. 2 (decode) in
hand-written CUDA; this package is only its ctypes binding (rotatek.py).
"""
from .rotatek import (calibrate, calibrate_subspace, compress_kv, decode_attn, decode_attn_partial,  # noqa: F401
                      merge_partials, gather_tokens, select_topr, workspace, calib_state, calib_accumulate,
                      calibrate_from_state, state_doubles,
                      workspace_bytes, make_dims, lib, last_launch_count, debug_decode_trace, RotateKError,
                      BF16, F32, CENTER, QUERY_WEIGHT, EIG_FP64, EIG_TWOSIDED, SIMT_ONLY, DEFAULT_FLAGS,
                      OP_CALIBRATE, OP_DECODE, KERNEL_AUTO, KERNEL_GENERIC, KERNEL_FAST, KERNEL_GQA,
                      KERNEL_STEAL, DECODE_OVERLAP)
