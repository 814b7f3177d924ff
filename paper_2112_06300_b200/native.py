"""ctypes binding of lib/libccdk.so (the C ABI in include/ccdk.h).

There is no fallback: if the library is missing or no CUDA device is usable,
every call raises.  The library is built in-tree by build.py.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import abi
from .abi import P_F32, P_F64, P_U8, P_U16, P_U32, P_U64

LIB_PATH = os.environ.get("CCDK_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                     "libccdk.so")


class CcdkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[ccdk status {code}] {msg}")
        self.code = code


class InvalidInput(CcdkError, ValueError):
    """ccdkit::InvalidInput (core.hpp:47-53)."""


class ConfigError(CcdkError):
    """ccdkit::ConfigError (core.hpp:55-61)."""


class CapacityError(CcdkError):
    pass


_lib = None
_lock = threading.RLock()  # default_context() -> Context() -> lib() re-enters

_SIGS = {
    "ccdk_abi_version": (C.c_int, []),
    "ccdk_last_error": (C.c_char_p, []),
    "ccdk_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ccdk_ctx_destroy": (C.c_int, [C.c_void_p]),
    "ccdk_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ccdk_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "ccdk_ctx_set_interval_capacity": (C.c_int, [C.c_void_p, C.c_uint64]),
    "ccdk_round_reduced": (C.c_int, [C.c_void_p, P_F64, C.c_uint64, P_F32, P_F32]),
    "ccdk_build_boxes": (C.c_int, [C.c_void_p, P_F64, P_F64, C.c_uint64, P_U32, C.c_uint64, P_U32,
                                   C.c_uint64, C.c_double, P_F32, P_F32, P_U8, P_U32]),
    "ccdk_choose_axis": (C.c_int, [C.c_void_p, P_F32, P_F32, C.c_uint64, C.POINTER(C.c_int)]),
    "ccdk_broad_phase": (C.c_int, [C.c_void_p, C.c_int, P_F32, P_F32, P_U8, P_U32, C.c_uint64,
                                   C.c_uint64, P_U32, C.c_uint64, P_U32, C.c_uint64, C.c_uint64,
                                   C.c_uint64, P_U64, C.POINTER(abi.StqStats)]),
    "ccdk_fetch_pairs": (C.c_int, [C.c_void_p, P_U64]),
    "ccdk_fetch_round_sizes": (C.c_int, [C.c_void_p, P_U64]),
    "ccdk_classify": (C.c_int, [C.c_void_p, P_U64, C.c_uint64, P_F64, P_F64, C.c_uint64, P_U32,
                                C.c_uint64, P_U32, C.c_uint64, P_U8, P_F64, P_U64, P_U64, P_U64]),
    "ccdk_narrow_phase_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                           C.POINTER(abi.NarrowCfg), C.c_uint64, C.c_void_p, C.c_void_p,
                                           C.POINTER(abi.NarrowStats)]),
    "ccdk_broad_resident": (C.c_int, [C.c_void_p, C.POINTER(abi.PipelineCfg), C.c_uint32, C.c_uint32,
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_int), C.POINTER(C.c_float)]),
    "ccdk_copy_keys_device": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ccdk_ccd_keys_resident": (C.c_int, [C.c_void_p, C.POINTER(abi.PipelineCfg), C.c_void_p, C.c_uint64,
                                         C.c_int, C.POINTER(abi.Report)]),
    "ccdk_inclusion_boxes": (C.c_int, [C.c_void_p, P_U8, P_F64, P_F64, C.c_uint64, P_F64]),
    "ccdk_process_intervals": (C.c_int, [C.c_void_p, P_U8, P_F64, P_F64, P_U16, P_F64, P_F64,
                                         C.c_uint64, C.POINTER(abi.NarrowCfg), P_U8, P_F64, P_U8,
                                         P_F64, P_U16]),
    "ccdk_narrow_phase": (C.c_int, [C.c_void_p, P_U8, P_F64, P_F64, C.c_uint64,
                                    C.POINTER(abi.NarrowCfg), C.c_uint64, P_F64, P_U8,
                                    C.POINTER(abi.NarrowStats)]),
    "ccdk_ccd": (C.c_int, [C.c_void_p, P_F64, P_F64, C.c_uint64, P_U32, C.c_uint64, P_U32,
                           C.c_uint64, C.POINTER(abi.PipelineCfg), C.POINTER(abi.Report)]),
    "ccdk_ccd_into": (C.c_int, [C.c_void_p, P_F64, P_F64, C.c_uint64, P_U32, C.c_uint64, P_U32,
                                C.c_uint64, C.POINTER(abi.PipelineCfg), C.POINTER(abi.Report),
                                C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64),
                                C.c_void_p]),
    "ccdk_run_batched": (C.c_int, [C.c_void_p, P_F64, P_F64, C.c_uint64, P_U32, C.c_uint64, P_U32,
                                   C.c_uint64, P_F32, P_F32, P_U8, P_U32, C.c_uint64,
                                   C.POINTER(abi.PipelineCfg), C.POINTER(abi.Report), C.c_void_p,
                                   C.c_void_p]),  # sink: a ccdk_pairs_sink or None
    "ccdk_ccd_no_zero_toi": (C.c_int, [C.c_void_p, P_F64, P_F64, C.c_uint64, P_U32, C.c_uint64, P_U32,
                                       C.c_uint64, C.POINTER(abi.PipelineCfg), C.POINTER(abi.Report)]),
    "ccdk_query_min_separations": (C.c_int, [C.c_void_p, P_U8, P_F64, C.c_uint64,
                                             C.POINTER(abi.PipelineCfg), P_F64]),
    "ccdk_scene_upload": (C.c_int, [C.c_void_p, P_F64, P_F64, C.c_uint64, P_U32, C.c_uint64, P_U32,
                                    C.c_uint64]),
    "ccdk_ccd_resident": (C.c_int, [C.c_void_p, C.POINTER(abi.PipelineCfg), C.c_uint32, C.c_uint32,
                                    C.POINTER(abi.Report)]),
    "ccdk_last_toi_device_ptr": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "ccdk_copy_last_toi": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ccdk_fetch_query_results": (C.c_int, [C.c_void_p, P_F64, P_U8]),
}


def exported_symbols():
    return list(_SIGS)


def lib():
    """Load libccdk.so (fails loudly when it is missing: no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2112_06300_b200.build` "
                                      "(the CCD path has no CPU fallback)")
                L = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    f = getattr(L, name)
                    f.restype = res
                    f.argtypes = args
                if L.ccdk_abi_version() != 2:
                    raise ImportError("libccdk.so ABI version mismatch")
                _lib = L
    return _lib


def check(rc: int):
    if rc == abi.OK:
        return
    msg = lib().ccdk_last_error().decode(errors="replace")
    cls = {abi.INVALID_INPUT: InvalidInput, abi.CONFIG: ConfigError,
           abi.CAPACITY: CapacityError}.get(rc, CcdkError)
    raise cls(rc, msg)


class Context:
    """One device context (streams and grow-only device buffers).  Calls are
    serialised by a mutex inside the library; ``lock`` is held by the Python
    API across a produce-then-fetch sequence (e.g. ccd then its candidate
    pairs), so one context can be shared by threads like the reference's
    reentrant functions."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().ccdk_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self.lock = threading.RLock()

    def close(self):
        if self.h:
            lib().ccdk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        check(lib().ccdk_ctx_set_stream(self.h, C.c_void_p(stream_handle or 0) if stream_handle else None))

    def set_interval_capacity(self, n: int):
        check(lib().ccdk_ctx_set_interval_capacity(self.h, n))

    def synchronize(self):
        check(lib().ccdk_ctx_synchronize(self.h))


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        with _lock:
            if device not in _default:
                _default[device] = Context(device)
    return _default[device]


def p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def f64(a):
    return np.ascontiguousarray(a, np.float64)


def f32(a):
    return np.ascontiguousarray(a, np.float32)


def u8(a):
    return np.ascontiguousarray(a, np.uint8)


def u16(a):
    return np.ascontiguousarray(a, np.uint16)


def u32(a):
    return np.ascontiguousarray(a, np.uint32)


def u64(a):
    return np.ascontiguousarray(a, np.uint64)
