"""ctypes binding of libedl_b200.so (the C ABI declared in include/edl_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile).  There is
no fallback: if the library is missing every product entry point raises, so a GPU run can
never silently route through a CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EDL_LIB_PATH") or os.path.join(_HERE, "libedl_b200.so")

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
EDL_NO_CHECKPOINT = 15

STATUS_NAMES = {
    0: "Ok", 1: "Retry", 2: "Invalid", 3: "PeerGone", 4: "Timeout", 5: "VersionMismatch",
    6: "UnknownWorker", 7: "StaleShard", 8: "ShapeMismatch", 9: "OutOfRange", 10: "CudaError",
    11: "OutOfMemory", 12: "AllowanceExceeded", 13: "IOError", 14: "Truncated",
    15: "NoCheckpoint",
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


class EdlPartitionMeta(C.Structure):
    _fields_ = [("index", C.c_uint32), ("offset", C.c_uint64), ("length", C.c_uint64)]


class EdlNextShard(C.Structure):
    _fields_ = [("kind", C.c_int32), ("meta", EdlPartitionMeta), ("resume_offset", C.c_uint64),
                ("epoch", C.c_uint64)]


class EdlSyntheticSpec(C.Structure):
    _fields_ = [("size", C.c_uint64), ("dim", C.c_int32), ("seed", C.c_uint64),
                ("noise", C.c_double), ("sign_labels", C.c_int32)]


class EdlRun(C.Structure):
    _fields_ = [("first", C.c_uint64), ("count", C.c_uint64)]


class EdlJobConfig(C.Structure):
    _fields_ = [("model", C.c_int32), ("data", EdlSyntheticSpec), ("num_classes", C.c_int32),
                ("layers", C.c_int32), ("hidden", C.c_int32), ("eta", C.c_double),
                ("decay", C.c_double), ("momentum", C.c_double), ("batch", C.c_int64),
                ("per_worker_batch", C.c_int64), ("lease_seed", C.c_uint64),
                ("partitions", C.c_int32), ("max_workers", C.c_int32), ("init_seed", C.c_uint64),
                ("t_a_ms", C.c_double), ("keep_log", C.c_int32), ("dry_run", C.c_int32),
                ("appx_recovery", C.c_int32)]


class EdlRecovery(C.Structure):
    _fields_ = [("mode", C.c_int32), ("status", C.c_int32), ("t_resume", C.c_uint64),
                ("version", C.c_uint64)]


class EdlStepReport(C.Structure):
    _fields_ = [("t", C.c_uint64), ("version", C.c_uint64), ("ring_size", C.c_int32),
                ("switched", C.c_int32), ("count", C.c_uint64), ("loss", C.c_double),
                ("step_ms", C.c_double), ("stall_ms", C.c_double)]


def _declare(L: C.CDLL) -> None:
    i32, i64, u32, u64, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    vp, sz, cp = C.c_void_p, C.c_size_t, C.c_char_p
    P = C.POINTER
    cpp = P(C.c_char_p)
    ci = C.c_int
    sig = {
        "edl_last_error": ([], cp), "edl_version": ([], cp),
        "edl_gemm_bf16": ([vp, i32, i32, vp, i32, i32, vp, i32, i32, i32, i32, i32, i32, vp, i32,
                           i32, vp], ci),
        "edl_default_partition_count": ([i32], i32),
        "edl_lease_create": ([u64, i32, u64, cp, P(vp)], ci),
        "edl_lease_destroy": ([vp], None),
        "edl_lease_register": ([vp, cp], ci), "edl_lease_unregister": ([vp, cp], ci),
        "edl_lease_is_registered": ([vp, cp], ci),
        "edl_lease_next": ([vp, cp, P(EdlNextShard)], ci),
        "edl_lease_report": ([vp, cp, u32, u64], ci),
        "edl_lease_reclaim": ([vp, cp], ci),
        "edl_lease_reclaim_at": ([vp, cp, P(u32), P(u64), sz], ci),
        "edl_lease_reclaim_missing": ([vp, cpp, sz], ci),
        "edl_lease_partition_meta": ([vp, u32, P(EdlPartitionMeta)], ci),
        "edl_lease_worker_shards": ([vp, cp, P(u32), P(u64), sz], sz),
        "edl_lease_snapshot": ([vp, vp, sz, P(sz)], ci),
        "edl_lease_restore": ([vp, vp, sz], ci),
        "edl_lease_epoch": ([vp], u64), "edl_lease_epochs_completed": ([vp], u64),
        "edl_lease_cursor": ([vp], u64), "edl_lease_permutation": ([vp, P(u32), sz], sz),
        "edl_lease_reclaimed_count": ([vp], sz), "edl_lease_in_flight_count": ([vp], sz),
        "edl_split_batch": ([i64, i32, P(i64)], ci),
        "edl_switch_delay": ([f64, f64], i64),
        "edl_eta_at": ([f64, f64, u64], f64),
        "edl_dataset_create_synthetic": ([P(EdlSyntheticSpec), i32, i32, P(vp)], ci),
        "edl_dataset_destroy": ([vp], None),
        "edl_dataset_size": ([vp], u64), "edl_dataset_dim": ([vp], i32),
        "edl_dataset_features": ([vp], vp), "edl_dataset_labels": ([vp], vp),
        "edl_dataset_true_weights": ([vp, P(f64)], ci),
        "edl_dataset_get": ([vp, u64, P(f64), P(f64)], ci),
        "edl_gather": ([vp, vp, i32, i64, vp, vp, vp], ci),
        "edl_local_gradient": ([i32, vp, vp, vp, i64, i32, vp, vp], ci),
        "edl_batch_loss": ([i32, vp, vp, vp, i64, i32, vp, vp], ci),
        "edl_sgd_step": ([vp, vp, i64, f64, i32, vp], ci),
        "edl_ring_allreduce_f64": ([P(vp), i32, sz, i32, vp, vp], ci),
        "edl_job_config_default": ([P(EdlJobConfig)], None),
        "edl_job_create": ([P(EdlJobConfig), cpp, P(i32), i32, P(vp)], ci),
        "edl_job_create_joining": ([P(EdlJobConfig), cpp, i32, cpp, i32, cp, i32, i32, i64, P(vp)],
                                   ci),
        "edl_job_destroy": ([vp], None),
        "edl_job_step": ([vp, P(EdlStepReport)], ci),
        "edl_job_sync": ([vp, P(EdlStepReport)], ci),
        "edl_job_scale_out": ([vp, cpp, P(i32), i32, P(i64)], ci),
        "edl_job_scale_in": ([vp, cpp, i32, f64, P(i64)], ci),
        "edl_job_schedule": ([vp, i64, i32, cpp, P(i32), i32], ci),
        "edl_job_params": ([vp, cp, vp, sz], ci),
        "edl_job_param_count": ([vp], sz),
        "edl_job_t": ([vp], u64),
        "edl_job_median_step_ms": ([vp], f64),
        "edl_job_log": ([vp, vp, sz, P(sz)], ci),
        "edl_job_ring": ([vp, vp, sz, P(sz)], ci),
        "edl_job_lease_snapshot": ([vp, vp, sz, P(sz)], ci),
        "edl_job_stream": ([vp], vp),
        "edl_job_set_profile": ([vp, i32], None),
        "edl_job_exchange_mode": ([vp], ci),
        "edl_job_join": ([vp], ci),
        "edl_job_counters": ([vp, P(f64), P(u64), P(u64)], None),
        "edl_job_reset_counters": ([vp], None),
        "edl_job_export": ([vp, vp, sz, P(sz)], ci),
        "edl_job_import": ([vp, vp, sz], ci),
        "edl_job_export_state": ([vp, vp, sz, P(sz)], ci),
        "edl_job_adopt_state": ([vp, vp, sz, i64], ci),
        "edl_job_gather_master": ([vp], ci),
        "edl_job_set_params": ([vp, vp, sz], ci),
        "edl_gemm_wgrad_sgd": ([vp, i32, vp, i32, vp, vp, i32, i32, i32, i32, C.c_float, vp], ci),
        "edl_gemm_wgrad_sgd_split": ([vp, i32, vp, i32, vp, vp, vp, i32, i32, i32, i32, i32, C.c_float, vp], ci),
        "edl_master_split": ([vp, vp, vp, C.c_size_t, vp], ci),
        "edl_master_join": ([vp, vp, vp, C.c_size_t, vp], ci),
        "edl_detect_straggler": ([P(f64), i32, i32, i32, f64, P(i32)], ci),
        "edl_job_save_checkpoint": ([vp, cp], ci),
        "edl_job_load_checkpoint": ([vp, cp], ci),
        "edl_job_fail": ([vp, cpp, i32, i32, P(EdlRecovery)], ci),
        "edl_job_worker_ms": ([vp, cp, P(f64), sz, P(sz)], ci),
        "edl_job_straggler": ([vp, i32, f64, vp, sz, P(sz)], ci),
        "edl_job_set_worker_delay": ([vp, cp, f64], ci),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)  # AttributeError = the library lacks a declared entry point
        fn.argtypes = args
        fn.restype = res
    for name, args, res in _EXTRA:
        if hasattr(L, name):
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res


HEADER_SYMBOLS = None  # filled lazily by exported_symbols()


def header_symbols() -> list:
    """Every function declared in include/edl_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "edl_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(edl_[a-z0-9_]+)\s*\(", text)))


def cstrs(items) -> "C.Array":
    arr = (C.c_char_p * max(1, len(items)))()
    for i, s in enumerate(items):
        arr[i] = s.encode()
    return arr


_EXTRA: list = []  # filled by modules that add entry points (see declare())


def declare(name: str, args: list, res=C.c_int) -> None:
    _EXTRA.append((name, args, res))
    if _lib is not None and hasattr(_lib, name):
        fn = getattr(_lib, name)
        fn.argtypes = args
        fn.restype = res
