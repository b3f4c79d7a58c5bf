"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference EDL hot path (liboracle.so, prefix ``or_``) and, when it has
been built in this container, the reference's own code compiled from /root/reference
(_ref/libedlref.so, prefix ``ref_``).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package — and only as the checker or
the timed CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libedlref.so")


def build(ref: bool | None = None) -> None:
    """make liboracle.so; also _ref/libedlref.so when /root/reference is present."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])
    if ref is None:
        ref = os.path.isdir("/root/reference/proj/src")
    if ref:
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


class Native:
    """ctypes view of one C API flavour (restated ``or`` or reference ``ref``)."""

    def __init__(self, path: str, prefix: str):
        self.lib = C.CDLL(path)
        self.prefix = prefix
        i32, i64, u32, u64, f64 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
        vp, sz, cp = C.c_void_p, C.c_size_t, C.c_char_p
        P = C.POINTER
        sig = {
            "synth_get": ([u64, C.c_int, u64, f64, C.c_int, u64, P(f64), P(f64)], C.c_int),
            "synth_true_weights": ([u64, C.c_int, u64, f64, C.c_int, P(f64)], C.c_int),
            "lease_create": ([u64, C.c_int, u64, cp], vp),
            "lease_destroy": ([vp], None),
            "lease_register": ([vp, cp], None),
            "lease_unregister": ([vp, cp], None),
            "lease_is_registered": ([vp, cp], C.c_int),
            "lease_next": ([vp, cp, P(C.c_int), P(u32), P(u64), P(u64), P(u64), P(u64)], C.c_int),
            "lease_report": ([vp, cp, u32, u64], C.c_int),
            "lease_reclaim": ([vp, cp], None),
            "lease_reclaim_at": ([vp, cp, P(u32), P(u64), sz], None),
            "lease_reclaim_missing": ([vp, cp], None),
            "lease_meta": ([vp, u32, P(u64), P(u64)], None),
            "lease_worker_shards": ([vp, cp, P(u32), P(u64), sz], sz),
            "lease_snapshot": ([vp, vp, sz], sz),
            "lease_restore": ([vp, vp, sz], C.c_int),
            "lease_epoch": ([vp], u64),
            "lease_epochs_completed": ([vp], u64),
            "lease_cursor": ([vp], u64),
            "lease_permutation": ([vp, P(u32), sz], sz),
            "lease_reclaimed_count": ([vp], sz),
            "lease_in_flight_count": ([vp], sz),
            "local_gradient": ([C.c_int, P(f64), C.c_int, P(f64), P(f64), i64, P(f64)], C.c_int),
            "batch_loss": ([C.c_int, P(f64), C.c_int, P(f64), P(f64), i64], f64),
            "sgd_step": ([P(f64), P(f64), C.c_int, u64, f64], C.c_int),
            "ring_reduce": ([P(f64), C.c_int, sz, C.c_int, P(f64)], C.c_int),
            "check_coverage": ([cp, u64, P(u64), C.c_char_p, sz], C.c_int),
            "replay": ([cp, C.c_int, u64, C.c_int, u64, f64, C.c_int, P(f64), f64, f64, C.c_int,
                        P(f64), P(u64), C.c_char_p, sz], C.c_int),
            "job_create": ([u64, C.c_int, u64, f64, C.c_int, C.c_int, f64, f64, i64, i64, u64,
                            C.c_int, cp, P(f64)], vp),
            "job_destroy": ([vp], None),
            "job_schedule": ([vp, i64, C.c_int, cp], None),
            "job_step": ([vp, P(f64), P(u64)], C.c_int),
            "job_params": ([vp, P(f64)], C.c_int),
            "job_t": ([vp], u64),
            "job_ring_size": ([vp], C.c_int),
            "job_plan": ([vp, C.c_int, C.c_char_p, sz, P(u64), P(u64), sz, P(sz)], C.c_int),
            "job_log_text": ([vp, C.c_char_p, sz, P(sz)], C.c_int),
            "job_snapshot": ([vp], vp),
            "job_snap_free": ([vp, vp], None),
            "job_restore": ([vp, vp, cp], None),
            "job_fail_approximate": ([vp, cp], None),
            "split_batch": ([i64, C.c_int, P(i64)], C.c_int),
            "switch_delay": ([f64, f64], i64),
            "eta_at": ([f64, f64, u64], f64),
            "default_partition_count": ([C.c_int], C.c_int),
            "ring_allreduce_threads": ([P(f64), C.c_int, sz, P(f64)], C.c_int),
        }
        for name, (args, res) in sig.items():
            full = f"{prefix}_{name}"
            if hasattr(self.lib, full):
                fn = getattr(self.lib, full)
                fn.argtypes = args
                fn.restype = res
                setattr(self, name, fn)


_cache: dict = {}


def restated() -> Native:
    if "or" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _cache["or"] = Native(ORACLE_SO, "or")
    return _cache["or"]


def reference() -> Native | None:
    """The reference compiled from its own sources, or None when not built here."""
    if "ref" not in _cache:
        _cache["ref"] = Native(REF_SO, "ref") if os.path.exists(REF_SO) else None
    return _cache["ref"]
