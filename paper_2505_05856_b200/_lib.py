"""ctypes binding of include/dawnpiper.h (the extension's C ABI).

There is no fallback: if the in-tree `_dawnpiper.so` is missing or the device
is not sm_100, `lib()` raises and every product path fails loudly.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

SO_PATH = Path(__file__).resolve().parent / "_dawnpiper.so"

_i64, _i32, _f32, _vp = C.c_int64, C.c_int32, C.c_float, C.c_void_p
_fp = C.POINTER(C.c_float)


class GemmArgs(C.Structure):
    _fields_ = [
        ("M", _i64), ("N", _i64), ("K", _i64),
        ("batch1", _i64), ("batch2", _i64),
        ("A", _vp), ("lda", _i64), ("a_s1", _i64), ("a_s2", _i64), ("a_mn_major", _i32),
        ("B", _vp), ("ldb", _i64), ("b_s1", _i64), ("b_s2", _i64), ("b_mn_major", _i32),
        ("C", _vp), ("ldc", _i64), ("c_s1", _i64), ("c_s2", _i64), ("c_dtype", _i32),
        ("accumulate", _i32),
        ("bias", _vp),
        ("residual", _vp), ("ldr", _i64), ("r_s1", _i64), ("r_s2", _i64),
        ("residual_mode", _i32),
        ("aux", _vp),
        ("alpha", _f32), ("gelu", _i32),
        ("block_n", _i32),
        ("split_k", _i32),
        ("cta_group", _i32),
        ("epilogue", _i32),
        ("colsum", _vp),
    ]


# name -> argtypes (all return c_int)
SIGNATURES = {
    "dpn_version": [],
    "dpn_init": [C.c_int],
    "dpn_host_alloc": [_i64, C.POINTER(_vp)],
    "dpn_host_free": [_vp],
    "dpn_memset_async": [_vp, C.c_int, _i64, _vp],
    "dpn_arena_create": [C.c_int, _i64, C.POINTER(C.c_int)],
    "dpn_arena_destroy": [C.c_int],
    "dpn_arena_select": [C.c_int],
    "dpn_arena_stats": [C.c_int, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64)],
    "dpn_arena_reset_peak": [C.c_int],
    "dpn_destroy": [],
    "dpn_swap_out": [_vp, _vp, _i64, _vp, _vp, _vp],
    "dpn_swap_in": [_vp, _vp, _i64, _vp, _vp, _vp],
    "dpn_p2p_copy": [_vp, C.c_int, _vp, C.c_int, _i64, _vp],
    "dpn_enable_peer": [C.c_int, C.c_int],
    "dpn_gemm": [C.POINTER(GemmArgs), _vp],
    "dpn_attn_fwd": [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _f32, C.c_int, _vp],
    "dpn_attn_bwd": [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _f32, C.c_int, _vp, _vp],
    "dpn_attn_fwd_cross": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _f32, _vp],
    "dpn_attn_bwd_cross": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64,
                           _f32, _vp],
    "dpn_layernorm_fwd": [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _vp],
    "dpn_layernorm_bwd": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _i64, _vp],
    "dpn_layernorm_bwd_fused": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp],
    "dpn_softmax_fwd": [_vp, _vp, _i64, _i64, _i64, _f32, C.c_int, _vp],
    "dpn_softmax_bwd": [_vp, _vp, _vp, _i64, _i64, _f32, _vp],
    "dpn_gelu_fwd": [_vp, _vp, _i64, _vp],
    "dpn_gelu_bwd": [_vp, _vp, _vp, _i64, _vp],
    "dpn_add": [_vp, _vp, _vp, _i64, _vp],
    "dpn_cast_f32_bf16": [_vp, _vp, _i64, _vp],
    "dpn_colsum": [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp],
    "dpn_xent": [_vp, _i64, _vp, _i64, _i64, _f32, _f32, _vp, _vp, _vp],
    "dpn_embed_fwd": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp],
    "dpn_embed_bwd": [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp],
    "dpn_adamw": [_vp, _vp, _vp, _vp, _vp, _i64, _f32, _f32, _f32, _f32, _f32, _i64, _vp],
    "dpn_adamw_dstep": [_vp, _vp, _vp, _vp, _vp, _i64, _f32, _f32, _f32, _f32, _f32, _vp, _vp],
    "dpn_relu_fwd": [_vp, _vp, _i64, _vp],
    "dpn_relu_bwd": [_vp, _vp, _vp, _i64, _vp],
    "dpn_dwconv3_fwd": [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp],
    "dpn_dwconv3_bwd": [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp],
    "dpn_bn_fwd": [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _vp],
    "dpn_bn_bwd": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _f32, _vp],
    "dpn_pool3_fwd": [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, C.c_int, _vp],
    "dpn_pool3_bwd": [_vp, _vp, _vp, _i64, _i64, _i64, _i64, _i64, C.c_int, _vp],
    "dpn_copy_cols": [_vp, _i64, _vp, _i64, _i64, _i64, C.c_int, _vp],
    "dpn_im2col3": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp],
    "dpn_gap_fwd": [_vp, _vp, _i64, _i64, _i64, _vp],
    "dpn_gap_bwd": [_vp, _vp, _i64, _i64, _i64, _vp],
}

_lock = threading.Lock()
_lib = None


class DpnError(RuntimeError):
    pass


def load_library() -> C.CDLL:
    """Load and type the shared library (no device needed)."""
    global _lib
    with _lock:
        if _lib is None:
            if not SO_PATH.exists():
                raise DpnError(f"CUDA extension not built: {SO_PATH} missing "
                               "(run `python -m paper_2505_05856_b200.build`)")
            lib = C.CDLL(str(SO_PATH))
            for name, argt in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argt
                fn.restype = C.c_int
            lib.dpn_last_error.argtypes = []
            lib.dpn_last_error.restype = C.c_char_p
            # torch's pluggable-allocator entry points (called by torch, typed for completeness)
            lib.dpn_arena_malloc.argtypes = [C.c_size_t, C.c_int, _vp]
            lib.dpn_arena_malloc.restype = _vp
            lib.dpn_arena_free.argtypes = [_vp, C.c_size_t, C.c_int, _vp]
            lib.dpn_arena_free.restype = None
            _lib = lib
    return _lib


def lib() -> C.CDLL:
    return load_library()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().dpn_last_error().decode(errors="replace")
        raise DpnError(f"{what or 'dpn call'} failed (rc={rc}): {msg}")


_inited = set()


def init_device(device: int) -> None:
    if device not in _inited:
        check(lib().dpn_init(device), "dpn_init")
        _inited.add(device)
