"""Partition leasing — host mirror of edl::ShardManager.

Same names, argument meaning and error behaviour as include/edl/datapipeline.hpp:23-127 of the
reference; the state machine runs in libedl_b200.so (csrc/lease.cpp) and is bit-compatible
with the reference (permutation stream, hand-out order, snapshot bytes).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum

from . import _lib


class PipeStatus(IntEnum):  # datapipeline.hpp:53
    Ok = 0
    UnknownWorker = 6
    StaleShard = 7
    ShapeMismatch = 8


@dataclass(frozen=True)
class PartitionMeta:  # datapipeline.hpp:23-29
    index: int
    locator: str
    offset: int
    length: int


@dataclass(frozen=True)
class ProgressRecord:  # datapipeline.hpp:31-35
    worker: str
    partition: int
    next_sample_offset: int


@dataclass(frozen=True)
class Shard:  # datapipeline.hpp:37-40
    meta: PartitionMeta
    resume_offset: int = 0


@dataclass(frozen=True)
class EpochEnd:  # datapipeline.hpp:42-44
    epoch: int


@dataclass(frozen=True)
class ShardPending:  # datapipeline.hpp:49
    pass


@dataclass(frozen=True)
class NextResult:  # ShardManager::NextResult, datapipeline.hpp:70-73
    status: PipeStatus
    value: object


def default_partition_count(max_expected_workers: int) -> int:  # datapipeline.cpp:9-11
    return _lib.lib().edl_default_partition_count(max_expected_workers)


class ShardManager:
    """Leader-owned dynamic data assignment (datapipeline.hpp:58)."""

    def __init__(self, dataset_size: int, partitions: int, seed: int, locator: str = ""):
        self._L = _lib.lib()
        h = C.c_void_p()
        _lib.check(self._L.edl_lease_create(dataset_size, partitions, seed, locator.encode(),
                                            C.byref(h)))
        self._h = h
        self._locator = locator

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.edl_lease_destroy(self._h)
            self._h = None

    def register_worker(self, worker: str) -> None:
        _lib.check(self._L.edl_lease_register(self._h, worker.encode()))

    def unregister_worker(self, worker: str) -> None:
        _lib.check(self._L.edl_lease_unregister(self._h, worker.encode()))

    def is_registered(self, worker: str) -> bool:
        return bool(self._L.edl_lease_is_registered(self._h, worker.encode()))

    def _meta(self, m) -> PartitionMeta:
        return PartitionMeta(m.index, self._locator, m.offset, m.length)

    def next_shard(self, worker: str) -> NextResult:
        out = _lib.EdlNextShard()
        rc = self._L.edl_lease_next(self._h, worker.encode(), C.byref(out))
        if rc == PipeStatus.UnknownWorker:
            return NextResult(PipeStatus.UnknownWorker, ShardPending())
        _lib.check(rc)
        if out.kind == 0:
            return NextResult(PipeStatus.Ok, Shard(self._meta(out.meta), out.resume_offset))
        if out.kind == 1:
            return NextResult(PipeStatus.Ok, EpochEnd(out.epoch))
        return NextResult(PipeStatus.Ok, ShardPending())

    def report_progress(self, rec: ProgressRecord) -> PipeStatus:
        rc = self._L.edl_lease_report(self._h, rec.worker.encode(), rec.partition,
                                      rec.next_sample_offset)
        if rc in (PipeStatus.UnknownWorker, PipeStatus.StaleShard):
            return PipeStatus(rc)
        _lib.check(rc)
        return PipeStatus.Ok

    def reclaim(self, worker: str) -> None:
        _lib.check(self._L.edl_lease_reclaim(self._h, worker.encode()))

    def reclaim_at(self, worker: str, offsets) -> None:
        offsets = list(offsets)
        ps = (C.c_uint32 * max(1, len(offsets)))(*[p for p, _ in offsets])
        os_ = (C.c_uint64 * max(1, len(offsets)))(*[o for _, o in offsets])
        _lib.check(self._L.edl_lease_reclaim_at(self._h, worker.encode(), ps, os_, len(offsets)))

    def reclaim_missing(self, live) -> None:
        live = sorted(live)
        _lib.check(self._L.edl_lease_reclaim_missing(self._h, _lib.cstrs(live), len(live)))

    def partition_meta(self, index: int) -> PartitionMeta:
        m = _lib.EdlPartitionMeta()
        _lib.check(self._L.edl_lease_partition_meta(self._h, index, C.byref(m)))
        return self._meta(m)

    def worker_shards(self, worker: str):
        n = self._L.edl_lease_worker_shards(self._h, worker.encode(), None, None, 0)
        ps = (C.c_uint32 * max(1, n))()
        os_ = (C.c_uint64 * max(1, n))()
        self._L.edl_lease_worker_shards(self._h, worker.encode(), ps, os_, n)
        return [(ps[i], os_[i]) for i in range(n)]

    def snapshot(self) -> bytes:
        n = C.c_size_t()
        _lib.check(self._L.edl_lease_snapshot(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        _lib.check(self._L.edl_lease_snapshot(self._h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def restore(self, snap: bytes) -> PipeStatus:
        buf = (C.c_uint8 * max(1, len(snap))).from_buffer_copy(snap or b"\0")
        rc = self._L.edl_lease_restore(self._h, buf, len(snap))
        if rc == _lib.EDL_SHAPE_MISMATCH:
            return PipeStatus.ShapeMismatch
        _lib.check(rc)
        return PipeStatus.Ok

    def epoch(self) -> int:
        return self._L.edl_lease_epoch(self._h)

    def epochs_completed(self) -> int:
        return self._L.edl_lease_epochs_completed(self._h)

    def cursor(self) -> int:
        return self._L.edl_lease_cursor(self._h)

    def permutation(self) -> list:
        n = self._L.edl_lease_permutation(self._h, None, 0)
        out = (C.c_uint32 * max(1, n))()
        self._L.edl_lease_permutation(self._h, out, n)
        return list(out[:n])

    def reclaimed_count(self) -> int:
        return self._L.edl_lease_reclaimed_count(self._h)

    def in_flight_count(self) -> int:
        return self._L.edl_lease_in_flight_count(self._h)
