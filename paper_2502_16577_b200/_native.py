"""ctypes binding of libpk_b200.so (include/permkit_b200.h).

The library is built in-tree by ``python -m paper_2502_16577_b200.build``
(or ``__graft_entry__.build()``). Loading it is mandatory: there is no CPU
fallback, so a missing library or device raises DeviceError. ctypes drops
the GIL around every foreign call, which lets several host threads drive
several devices at once, like permkit's thread-pool executor
(parallel.py:333-341).
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Sequence

import numpy as np

from .errors import DeviceError, ImpossibleError, PolicyError, StructureError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PK_B200_LIB", os.path.join(_HERE, "libpk_b200.so"))

PK_OK = 0
PK_ERR_ARG = 1
PK_ERR_POLICY = 2
PK_ERR_STRUCTURE = 3
PK_ERR_IMPOSSIBLE = 4
PK_ERR_CUDA = 5
PK_ERR_OVERFLOW = 6

PK_FLAG_EXACT = 1
PK_FLAG_SPARSE = 2
PK_FLAG_PRECISE = 4


class RunStats(ctypes.Structure):
    _fields_ = [
        ("kernel_ms", ctypes.c_double),
        ("wall_ms", ctypes.c_double),
        ("iterates", ctypes.c_uint64),
        ("chunks", ctypes.c_uint64),
        ("walker_ranges", ctypes.c_uint64),
        ("log2_chunk", ctypes.c_int32),
        ("devices", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


_lib = None
_lock = threading.Lock()


class DecompStats_(ctypes.Structure):
    _fields_ = [("tasks_created", ctypes.c_uint64), ("d1_applied", ctypes.c_uint64),
                ("d2_applied", ctypes.c_uint64), ("d34_applied", ctypes.c_uint64),
                ("trivial_leaves", ctypes.c_uint64), ("kernel_leaves", ctypes.c_uint64),
                ("dense_kernel_leaves", ctypes.c_uint64), ("max_depth", ctypes.c_int64),
                ("elapsed_s", ctypes.c_double)]


class DecompResult(ctypes.Structure):
    _fields_ = [("stats", DecompStats_), ("trivial", ctypes.c_int64), ("leaves", ctypes.c_int64),
                ("leaf_values", ctypes.c_int64)]


PK_KIND_REAL, PK_KIND_COMPLEX, PK_KIND_INT = 0, 1, 2
PK_ERR_TIMEOUT = 7

_D = ctypes.POINTER(ctypes.c_double)
_U64 = ctypes.POINTER(ctypes.c_uint64)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); kept in one table so tests can check that the
# library exports every symbol the header declares
SIGNATURES = {
    "pk_abi_version": (ctypes.c_int, []),
    "pk_device_count": (ctypes.c_int, []),
    "pk_last_error": (ctypes.c_char_p, []),
    "pk_fp64_peak": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _D, _D]),
    "pk_dense_f64": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_int, ctypes.c_uint32, ctypes.c_int, _I32, ctypes.c_int,
                                    _D, ctypes.POINTER(RunStats)]),
    "pk_dense_f64_ranges": (ctypes.c_int, [_D, _D, ctypes.c_int, _U64, _U64, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, _D]),
    "pk_dense_f64_chunks": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                           ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                                           ctypes.c_int, _D, _D]),
    "pk_dense_c128": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_uint32, ctypes.c_int, _I32, ctypes.c_int, _D,
                                     ctypes.POINTER(RunStats)]),
    "pk_dense_c128_ranges": (ctypes.c_int, [_D, _D, ctypes.c_int, _U64, _U64, ctypes.c_int,
                                            ctypes.c_int, _D]),
    "pk_dense_c128_chunks": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, _D,
                                            _D]),
    "pk_dense_f64_batch": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_uint32, ctypes.c_int, _D,
                                          ctypes.POINTER(RunStats)]),
    "pk_sparse_f64": (ctypes.c_int, [_I64, _I64, _D, ctypes.c_int, _D, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                     _I32, ctypes.c_int, _D, ctypes.POINTER(RunStats)]),
    "pk_spa_f64_source": (ctypes.c_int, [_D, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                         ctypes.c_char_p, ctypes.c_uint64, _U64]),
    "pk_dense_c128_batch": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                           ctypes.c_int, _D, ctypes.POINTER(RunStats)]),
    "pk_sparse_c128": (ctypes.c_int, [_I64, _I64, _D, ctypes.c_int, _D, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, _I32,
                                      ctypes.c_int, _D, ctypes.POINTER(RunStats)]),
    "pk_spa_c128_source": (ctypes.c_int, [_D, ctypes.c_int, ctypes.c_uint32, ctypes.c_char_p,
                                          ctypes.c_uint64, _U64]),
    "pk_dd_accumulate": (ctypes.c_int, [_D, ctypes.c_int64, _D]),
    "pk_quantize_walk": (ctypes.c_int, [_D, _D, ctypes.c_int, ctypes.c_int, _D, _D]),
    "pk_decomp_tree": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
                                      ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                      ctypes.POINTER(ctypes.c_void_p),
                                      ctypes.POINTER(DecompResult)]),
    "pk_decomp_fetch": (ctypes.c_int, [ctypes.c_void_p, _I64, ctypes.c_void_p, _I64, _I32,
                                       ctypes.c_void_p, ctypes.c_void_p]),
    "pk_decomp_free": (None, [ctypes.c_void_p]),
    "pk_decomp_last_error": (ctypes.c_char_p, []),
    "pk_int": (ctypes.c_int, [_I64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                              ctypes.c_int, _I32, ctypes.c_int, _U64, ctypes.c_void_p,
                              ctypes.POINTER(RunStats)]),
    "pk_int_batch": (ctypes.c_int, [_I64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _U64,
                                    ctypes.c_void_p, ctypes.POINTER(RunStats)]),
    "pk_int_spa_source": (ctypes.c_int, [_I64, ctypes.c_int, ctypes.c_char_p, ctypes.c_uint64,
                                         _U64]),
    "pk_int_ranges": (ctypes.c_int, [_I64, ctypes.c_int, _U64, _U64, ctypes.c_int, ctypes.c_int,
                                     _U64, ctypes.c_void_p]),
}


def load(path: Optional[str] = None):
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise DeviceError(f"{p} is missing; build it with `python -m paper_2502_16577_b200.build`")
        try:
            lib = ctypes.CDLL(p)
        except OSError as exc:
            raise DeviceError(f"cannot load {p}: {exc}") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().pk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc == PK_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == PK_ERR_ARG:
        raise ValueError(msg)
    if rc == PK_ERR_POLICY:
        raise PolicyError(msg)
    if rc == PK_ERR_STRUCTURE:
        raise StructureError(msg)
    if rc == PK_ERR_IMPOSSIBLE:
        raise ImpossibleError(msg)
    if rc == PK_ERR_OVERFLOW:
        raise OverflowError(msg)
    raise DeviceError(msg)


def device_count() -> int:
    c = load().pk_device_count()
    if c < 0:
        raise DeviceError("cudaGetDeviceCount failed")
    return c


def fp64_peak_tflops(device: int = 0, iters: int = 20000) -> float:
    """Live DFMA throughput of `device` (the FP64 roofline denominator)."""
    tf = ctypes.c_double(0.0)
    ms = ctypes.c_double(0.0)
    rc = load().pk_fp64_peak(device, iters, ctypes.byref(tf), ctypes.byref(ms))
    check(rc, "pk_fp64_peak")
    return tf.value


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def u64ptr(a: np.ndarray):
    return a.ctypes.data_as(_U64)


def i32ptr(a: np.ndarray):
    return a.ctypes.data_as(_I32)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_I64)


def devices_arg(devices: Optional[Sequence[int]]):
    if not devices:
        return None, 0, None
    arr = np.ascontiguousarray(np.array(list(devices), dtype=np.int32))
    return i32ptr(arr), len(arr), arr  # keep arr alive
