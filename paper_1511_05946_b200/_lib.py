"""ctypes binding of ``libacdc_b200.so`` (the C ABI in ``include/acdc_b200.h``).

There is no fallback: if the library is missing or cannot be loaded, every
call raises.  Error codes map to the exception types the reference raises for
the same conditions (``ValueError`` for size/shape problems, ``RuntimeError``
for CUDA failures; transforms.py:96-97, layers.py:91-97).
"""

from __future__ import annotations

import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
# ACDC_LIB_PATH selects an alternative build of the same ABI (A/B kernel experiments)
LIB_PATH = os.environ.get("ACDC_LIB_PATH") or os.path.join(_PKG, "libacdc_b200.so")

ACDC_OK = 0
ACDC_E_SIZE = -1
ACDC_E_SHAPE = -2
ACDC_E_ALIGN = -3
ACDC_E_WS = -4
ACDC_E_CUDA = -5
ACDC_E_NULL = -6

ABI_VERSION = 1

class SgdStep(ctypes.Structure):
    """``acdc_sgd_step_t`` (include/acdc_b200.h): one momentum-SGD step of a, d, bias_d."""

    _fields_ = [
        ("value", ctypes.c_void_p * 3),
        ("velocity", ctypes.c_void_p * 3),
        ("lr", ctypes.c_float * 3),
        ("weight_decay", ctypes.c_float * 3),
        ("momentum", ctypes.c_float),
    ]


# name -> (restype, argtypes)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
SIGNATURES = {
    "acdc_abi_version": (ctypes.c_int, []),
    "acdc_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "acdc_last_error": (ctypes.c_char_p, []),
    "acdc_max_n": (ctypes.c_int, []),
    "acdc_prepare": (ctypes.c_int, [_I32]),
    "acdc_fwd_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I32, _I64, _I64, _P]),
    "acdc_bwd_workspace_bytes": (ctypes.c_size_t, [_I64, _I32]),
    "acdc_bwd_launch_count": (ctypes.c_int, [_I64, _I32, ctypes.c_int]),
    "acdc_bwd_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _I64, _I32, _I64, _I64, _I64, _P],
    ),
    "acdc_h2cache_bytes": (ctypes.c_size_t, [_I64, _I32]),
    "acdc_step_max_rows": (_I64, [_I32]),
    "acdc_step_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _I64, _I32, _I64, _I64, _I64, _I64, _P],
    ),
    "acdc_fwd_cache_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I32, _I64, _I64, _P]),
    "acdc_bwd_cached_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _I64, _I32, _I64, _I64, _I64, _P],
    ),
    "acdc_bwd_sgd_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, ctypes.c_int, _P, _P, _P, ctypes.c_int, ctypes.POINTER(SgdStep), _P, ctypes.c_size_t,
         _I64, _I32, _I64, _I64, _I64, _P],
    ),
    "acdc_dct2_f32": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _I64, _P]),
    "acdc_dct3_f32": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _I64, _P]),
    "cascade_ckpt_bytes": (ctypes.c_size_t, [_I64, _I32, _I32]),
    "cascade_fwd_f32": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "cascade_bwd_block_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _I64, _I32, _I64,
         _I64, _I64, _P],
    ),
    "afdf_fwd_c64": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _I64, _I64, _P]),
    "afdf_bwd_workspace_bytes": (ctypes.c_size_t, [_I64, _I32]),
    "afdf_bwd_c64": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _I64, _I32, _I64, _I64, _I64, _P],
    ),
    "acdc_fft_c64": (ctypes.c_int, [_P, _P, _I64, _I32, ctypes.c_int, _I64, _I64, _P]),
    "cascade_gather_supported": (ctypes.c_int, [_I32]),
    "cascade_bwd_block_gather_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _I64, _I32, _I64,
         _I64, _I64, _P],
    ),
    "cascade_defer_ws_bytes": (ctypes.c_size_t, [_I64, _I32]),
    "cascade_bwd_block_defer_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, ctypes.c_size_t, _I64, _I32, _I64, _I64, _I64, _P],
    ),
    "cascade_grad_reduce_f32": (ctypes.c_int, [_P, ctypes.c_size_t, _I32, _I64, _I32, _P, ctypes.c_int, _P]),
    "cascade_pair_supported": (ctypes.c_int, [_I64, _I32]),
    "cascade_hl_supported": (ctypes.c_int, [_I32]),
    "cascade_fwd_hl_f32": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "cascade_hl_defer_ws_bytes": (ctypes.c_size_t, [_I64, _I32]),
    "cascade_bwd_hl_defer_f32": (
        ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _I64, _I32, _I64, _I64, _I64, _P]),
    "cascade_grad_reduce_hl_f32": (ctypes.c_int, [_P, ctypes.c_size_t, _I32, _I64, _I32, _P, ctypes.c_int, _P]),
    "cascade_bwd_pair_defer_f32": (
        ctypes.c_int,
        [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_int, ctypes.c_int, _P, _P, ctypes.c_size_t, _I64,
         _I32, _I64, _I64, _I64, _I64, _P],
    ),
    "acdc_relu_fwd_f32": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _I64, _P]),
    "acdc_relu_bwd_f32": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I64, _I64, _I64, _P]),
    "acdc_gather_cols": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _I64, _I64, _P]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1511_05946_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        ver = lib.acdc_abi_version()
        if ver != ABI_VERSION:
            raise RuntimeError(f"libacdc_b200 ABI {ver} != expected {ABI_VERSION}")
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == ACDC_OK:
        return
    msg = load().acdc_strerror(rc).decode()
    if rc == ACDC_E_CUDA:
        raise RuntimeError(msg)
    raise ValueError(msg)
