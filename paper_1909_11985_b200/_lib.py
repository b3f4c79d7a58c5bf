"""ctypes binding of libedl_b200.so (the C ABI declared in include/edl_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile).  There is
no fallback: if the library is missing every product entry point raises, so a GPU run can
never silently route through a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libedl_b200.so")

EDL_OK = 0
EDL_RETRY = 1
EDL_EINVAL = 2
EDL_PEER_GONE = 3
EDL_TIMEOUT = 4
EDL_VERSION_MISMATCH = 5
EDL_UNKNOWN_WORKER = 6
EDL_STALE_SHARD = 7
EDL_SHAPE_MISMATCH = 8
EDL_OUT_OF_RANGE = 9
EDL_ECUDA = 10
EDL_ENOMEM = 11
EDL_ALLOWANCE_EXCEEDED = 12
EDL_EIO = 13
EDL_ETRUNCATED = 14

STATUS_NAMES = {
    0: "Ok", 1: "Retry", 2: "Invalid", 3: "PeerGone", 4: "Timeout", 5: "VersionMismatch",
    6: "UnknownWorker", 7: "StaleShard", 8: "ShapeMismatch", 9: "OutOfRange", 10: "CudaError",
    11: "OutOfMemory", 12: "AllowanceExceeded", 13: "IOError", 14: "Truncated",
}


class EdlError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def check(rc: int) -> int:
    if rc != EDL_OK:
        raise EdlError(rc, lib().edl_last_error().decode())
    return rc


def _declare(L: C.CDLL) -> None:
    i32, i64, u32, u64, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    vp, sz, cp = C.c_void_p, C.c_size_t, C.c_char_p
    L.edl_last_error.restype = cp
    L.edl_version.restype = cp
    L.edl_gemm_bf16.argtypes = [vp, i32, i32, vp, i32, i32, vp, i32, i32, i32, i32, i32, i32,
                                vp, i32, i32, vp]
    L.edl_gemm_bf16.restype = C.c_int
    for name, args, res in _EXTRA:
        if hasattr(L, name):
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res


_EXTRA: list = []  # filled by modules that add entry points (see declare())


def declare(name: str, args: list, res=C.c_int) -> None:
    _EXTRA.append((name, args, res))
    if _lib is not None and hasattr(_lib, name):
        fn = getattr(_lib, name)
        fn.argtypes = args
        fn.restype = res
