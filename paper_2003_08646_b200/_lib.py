"""ctypes binding of the C ABI in include/lance_b200.h.

The library is built in-tree (paper_2003_08646_b200/_build/liblance_b200.so)
by ``paper_2003_08646_b200.build``.  There is no fallback: if the library is
missing or no sm_100 device is present every call fails loudly.
"""
from __future__ import annotations

import ctypes as ct
import os
import threading

from . import build as _build

LIB_PATH = os.environ.get("LANCE_LIB_PATH", _build.LIB)  # override: A/B experiments only

LANCE_OK = 0
LANCE_ERR_INVALID_ARGUMENT = 1
LANCE_ERR_NAN = 2
LANCE_ERR_CUDA = 3
LANCE_ERR_NO_DEVICE = 4

DBG_CODES_A, DBG_ROWSUM, DBG_CODES_W, DBG_COLSUM = 1, 2, 3, 4


class CSpec(ct.Structure):
    _fields_ = [(n, ct.c_int) for n in ("n", "c", "h", "w", "k", "pad")]


class CConfig(ct.Structure):
    _fields_ = [(n, ct.c_int) for n in ("bits_w", "bits_i", "granularity", "mode")]


class CQParams(ct.Structure):
    _fields_ = [("bits", ct.c_int), ("t_min", ct.c_float), ("t_max", ct.c_float),
                ("scale", ct.c_float)]


_lock = threading.Lock()
_lib = None


def lib():
    """Load (building first if stale) the native library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            _build.build()
        L = ct.CDLL(LIB_PATH)
        P = ct.c_void_p
        L.lance_abi_version.restype = ct.c_int
        L.lance_status_string.restype = ct.c_char_p
        L.lance_status_string.argtypes = [ct.c_int]
        L.lance_last_error.restype = ct.c_char_p
        L.lance_validate.argtypes = [ct.POINTER(CSpec), ct.POINTER(CConfig)]
        L.lance_winograd_multiply_count.argtypes = [ct.POINTER(CSpec)]
        L.lance_winograd_multiply_count.restype = ct.c_uint64
        L.lance_direct_multiply_count.argtypes = [ct.POINTER(CSpec)]
        L.lance_direct_multiply_count.restype = ct.c_uint64
        L.lance_gemm_host.argtypes = [ct.POINTER(CSpec), ct.POINTER(CConfig), P, P, P]
        L.lance_host_cache_clear.argtypes = []
        L.lance_plan_create.argtypes = [ct.POINTER(CSpec), ct.POINTER(CConfig), ct.c_int,
                                        ct.POINTER(P)]
        L.lance_plan_destroy.argtypes = [P]
        L.lance_plan_device_bytes.argtypes = [P]
        L.lance_plan_device_bytes.restype = ct.c_size_t
        L.lance_plan_set_filters.argtypes = [P, P, P]
        L.lance_plan_forward.argtypes = [P, P, P, P]
        L.lance_plan_forward_static.argtypes = [P, ct.POINTER(CQParams), P, P, P]
        L.lance_plan_set_epilogue.argtypes = [P, P, ct.c_int]
        L.lance_plan_ranges.argtypes = [P, P, P, P]
        L.lance_plan_set_input_layout.argtypes = [P, ct.c_int]
        L.lance_plan_input_layout.argtypes = [P]
        L.lance_plan_set_epilogue_pool.argtypes = [P, ct.c_int]
        L.lance_plan_forward_ranges.argtypes = [P, P, P, P, P]
        L.lance_plan_sync.argtypes = [P, P]
        L.lance_plan_get_params.argtypes = [P, ct.POINTER(CQParams), ct.POINTER(CQParams)]
        L.lance_plan_debug_read.argtypes = [P, ct.c_int, P, ct.c_size_t]
        L.lance_plan_set_acc_dump.argtypes = [P, P]
        L.lance_plan_last_launch_count.argtypes = [P]
        L.lance_plan_stage_timing.argtypes = [P, ct.c_int]
        L.lance_plan_read_stage_times.argtypes = [P, ct.POINTER(ct.c_double),
                                                  ct.POINTER(ct.c_int)]
        L.lance_plan_create_tiled.argtypes = [ct.POINTER(CSpec), ct.POINTER(CConfig), ct.c_int,
                                              ct.c_int, ct.POINTER(P)]
        L.lance_plan_positions.argtypes = [P]
        L.lance_gemm_host_tiled.argtypes = [ct.POINTER(CSpec), ct.POINTER(CConfig), ct.c_int,
                                            P, P, P]
        L.lance_winograd_multiply_count_tiled.argtypes = [ct.POINTER(CSpec), ct.c_int]
        L.lance_winograd_multiply_count_tiled.restype = ct.c_uint64
        L.lance_maxpool2x2_nhwc.argtypes = [P, P, ct.c_int, ct.c_int, ct.c_int, ct.c_int, P]
        L.lance_fnv1a64.argtypes = [P, ct.c_size_t]
        L.lance_fnv1a64.restype = ct.c_uint64
        L.lance_uniform_fill.argtypes = [ct.c_uint64, P, ct.c_size_t]
        L.lance_uniform_fill.restype = None
        _lib = L
        return L


EXPORTED = [
    "lance_abi_version", "lance_status_string", "lance_last_error", "lance_validate",
    "lance_winograd_multiply_count", "lance_direct_multiply_count", "lance_gemm_host",
    "lance_host_cache_clear",
    "lance_plan_create", "lance_plan_destroy", "lance_plan_device_bytes",
    "lance_plan_set_filters", "lance_plan_forward", "lance_plan_forward_static",
    "lance_plan_set_epilogue", "lance_plan_ranges", "lance_plan_set_input_layout", "lance_plan_input_layout", "lance_plan_set_epilogue_pool", "lance_plan_forward_ranges", "lance_plan_sync", "lance_plan_get_params",
    "lance_plan_debug_read", "lance_plan_set_acc_dump", "lance_plan_last_launch_count",
    "lance_plan_stage_timing", "lance_plan_read_stage_times",
    "lance_plan_create_tiled", "lance_plan_positions", "lance_gemm_host_tiled",
    "lance_winograd_multiply_count_tiled", "lance_maxpool2x2_nhwc", "lance_fnv1a64",
    "lance_uniform_fill",
]
