"""ctypes loader for libtvprox.so (the C ABI in include/tvprox.h).

Argument marshalling only.  The product path has no fallback: if the shared
library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtvprox.so")

TVP_F32, TVP_F64 = 0, 1
LAM_SCALAR, LAM_PER_ROW, LAM_PER_EDGE, LAM_PER_CHANNEL, LAM_PER_PLANE = 0, 1, 2, 3, 4
TVP_OK, TVP_EINVAL, TVP_EUNSUPPORTED, TVP_ECUDA = 0, 1, 2, 3
ITERS_NOT_CONVERGED, ITERS_NONFINITE, ITERS_STALL_FLAG = -1, -2, 1 << 16
LS_BACKTRACK, LS_PARALLEL = 0, 1
HIST_BINS = 128


def iters_count(v):
    """PN iterations of a row_iters value >= 0 (bits 0..15)."""
    return v & 0xFFFF


def iters_ls(v):
    """Line-search passes of a row_iters value >= 0 (bits 20..27)."""
    return (v >> 20) & 0xFF


class Options(ctypes.Structure):
    """tvp_options_t (include/tvprox.h): per-call options of the *_ex entry points."""
    _fields_ = [("fused2d", ctypes.c_int), ("line_search", ctypes.c_int), ("ls_after", ctypes.c_int),
                ("diag", ctypes.c_void_p), ("iter_hist", ctypes.c_void_p)]

# every symbol include/tvprox.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "tvp_max_line", "tvp_max_line_1d", "tvp_set_fused2d", "tvp_options_default",
    "tv1d_mask_words", "tv1d_prox_fwd", "tv1d_prox_fwd_warm", "tv1d_prox_fwd_ex", "tv1d_bwd_workspace_bytes",
    "tv1d_prox_bwd",
    "tv2d_saved_bytes", "tv2d_workspace_bytes", "tv2d_prox_fwd", "tv2d_prox_bwd", "tv2d_prox_fwd_ex", "tv2d_prox_bwd_ex",
    "tv2d_lines_fwd", "tv2d_lines_workspace_bytes", "tv2d_lines_bwd",
    "tvp_softplus_fwd", "tvp_softplus_bwd", "tvp_axpby",
    "tvp_status_string", "tvp_last_error", "tvp_version", "tvp_launch_count",
]

_lock = threading.Lock()
_lib = None


class TVProxError(RuntimeError):
    pass


def _sig(lib, name, attr, value):
    """Type one entry point (an older library build lacking it is tolerated; calling it raises)."""
    fn = getattr(lib, name, None)
    if fn is not None:
        setattr(fn, attr, value)


def load(path: str = LIB_PATH):
    """Load and type the library (once)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise TVProxError(
                "libtvprox.so not found at %s: build it with `python -m paper_2204_03643_b200.build` "
                "(there is no CPU fallback)" % path)
        lib = ctypes.CDLL(path)
        i64, i32, u64 = ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
        vp, dbl = ctypes.c_void_p, ctypes.c_double
        _sig(lib, "tvp_max_line", "argtypes", [i32])
        _sig(lib, "tvp_max_line", "restype", i64)
        _sig(lib, "tvp_max_line_1d", "argtypes", [i32])
        _sig(lib, "tvp_set_fused2d", "argtypes", [i32])
        _sig(lib, "tvp_set_fused2d", "restype", i32)
        _sig(lib, "tvp_max_line_1d", "restype", i64)
        _sig(lib, "tv1d_mask_words", "argtypes", [i64])
        _sig(lib, "tv1d_mask_words", "restype", u64)
        _sig(lib, "tv1d_prox_fwd", "argtypes", [i32, vp, vp, i64, i64, i64, vp, i32, dbl, vp, vp, vp])
        _sig(lib, "tv1d_prox_fwd", "restype", i32)
        _sig(lib, "tv1d_prox_fwd_warm", "argtypes", [i32, vp, vp, i64, i64, i64, vp, i32, dbl, vp, vp, vp, vp])
        _sig(lib, "tv1d_prox_fwd_warm", "restype", i32)
        op = ctypes.POINTER(Options)
        _sig(lib, "tvp_options_default", "argtypes", [op])
        _sig(lib, "tvp_options_default", "restype", None)
        _sig(lib, "tv1d_prox_fwd_ex", "argtypes", [i32, vp, vp, i64, i64, i64, vp, i32, dbl, vp, vp, vp, op, vp])
        _sig(lib, "tv1d_prox_fwd_ex", "restype", i32)
        _sig(lib, "tv2d_prox_fwd_ex", "argtypes", [i32, vp, vp, i64, i64, i64, i64, vp, i32, dbl, i32, vp, vp, vp, op,
                                                   vp])
        _sig(lib, "tv2d_prox_fwd_ex", "restype", i32)
        _sig(lib, "tv2d_prox_bwd_ex", "argtypes", [i32, vp, vp, vp, vp, i64, i64, i64, i64, i32, i32, vp, op, vp])
        _sig(lib, "tv2d_prox_bwd_ex", "restype", i32)
        _sig(lib, "tv1d_bwd_workspace_bytes", "argtypes", [i32, i64, i32])
        _sig(lib, "tv1d_bwd_workspace_bytes", "restype", u64)
        _sig(lib, "tv1d_prox_bwd", "argtypes", [i32, vp, vp, vp, vp, i64, i64, i64, i32, vp, vp])
        _sig(lib, "tv1d_prox_bwd", "restype", i32)
        _sig(lib, "tv2d_saved_bytes", "argtypes", [i64, i64, i64, i64, i32])
        _sig(lib, "tv2d_saved_bytes", "restype", u64)
        _sig(lib, "tv2d_workspace_bytes", "argtypes", [i32, i64, i64, i64, i64, i32])
        _sig(lib, "tv2d_workspace_bytes", "restype", u64)
        _sig(lib, "tv2d_prox_fwd", "argtypes", [i32, vp, vp, i64, i64, i64, i64, vp, i32, dbl, i32, vp, vp, vp, vp])
        _sig(lib, "tv2d_prox_fwd", "restype", i32)
        _sig(lib, "tv2d_prox_bwd", "argtypes", [i32, vp, vp, vp, vp, i64, i64, i64, i64, i32, i32, vp, vp])
        _sig(lib, "tv2d_prox_bwd", "restype", i32)
        _sig(lib, "tv2d_lines_fwd", "argtypes", [i32, vp, vp, i64, i64, i64, i64, vp, i32, dbl, i32, vp, vp])
        _sig(lib, "tv2d_lines_fwd", "restype", i32)
        _sig(lib, "tv2d_lines_workspace_bytes", "argtypes", [i32, i64, i64, i64, i64, i32])
        _sig(lib, "tv2d_lines_workspace_bytes", "restype", u64)
        _sig(lib, "tv2d_lines_bwd", "argtypes", [i32, vp, vp, vp, vp, i64, i64, i64, i64, i32, i32, vp, vp])
        _sig(lib, "tv2d_lines_bwd", "restype", i32)
        _sig(lib, "tvp_softplus_fwd", "argtypes", [i32, vp, vp, i64, vp])
        _sig(lib, "tvp_softplus_fwd", "restype", i32)
        _sig(lib, "tvp_softplus_bwd", "argtypes", [i32, vp, vp, vp, i64, vp])
        _sig(lib, "tvp_softplus_bwd", "restype", i32)
        _sig(lib, "tvp_axpby", "argtypes", [i32, vp, vp, dbl, dbl, i64, vp])
        _sig(lib, "tvp_axpby", "restype", i32)
        _sig(lib, "tvp_status_string", "argtypes", [i32])
        _sig(lib, "tvp_status_string", "restype", ctypes.c_char_p)
        _sig(lib, "tvp_last_error", "argtypes", [])
        _sig(lib, "tvp_last_error", "restype", ctypes.c_char_p)
        _sig(lib, "tvp_version", "argtypes", [])
        _sig(lib, "tvp_version", "restype", i32)
        _sig(lib, "tvp_launch_count", "argtypes", [i32])
        _sig(lib, "tvp_launch_count", "restype", i64)
        _lib = lib
        return lib


def check(status: int, what: str):
    if status != TVP_OK:
        lib = load()
        msg = lib.tvp_last_error().decode(errors="replace")
        raise TVProxError("%s failed: %s (%s)" % (what, lib.tvp_status_string(status).decode(), msg))
