"""ORACLE — TEST INFRASTRUCTURE ONLY.  Pythonic wrappers over oracle.Native (or_/ref_)."""
from __future__ import annotations

import ctypes as C
import os
import tempfile

import numpy as np

from . import Native

P = C.POINTER
f64p = P(C.c_double)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(f64p)


def synth_get(nat: Native, spec: dict, index: int):
    feat = np.zeros(spec["dim"], dtype=np.float64)
    label = C.c_double()
    rc = nat.synth_get(spec["size"], spec["dim"], spec["seed"], spec.get("noise", 0.0),
                       int(spec.get("sign_labels", False)), index, _dp(feat), C.byref(label))
    return rc, feat, label.value


def true_weights(nat: Native, spec: dict) -> np.ndarray:
    w = np.zeros(spec["dim"], dtype=np.float64)
    nat.synth_true_weights(spec["size"], spec["dim"], spec["seed"], spec.get("noise", 0.0),
                           int(spec.get("sign_labels", False)), _dp(w))
    return w


class Leases:
    """ShardManager (datapipeline.hpp:58) through the oracle C API."""

    def __init__(self, nat: Native, size: int, d: int, seed: int, locator: str = ""):
        self.n = nat
        self.h = nat.lease_create(size, d, seed, locator.encode())

    def __del__(self):
        if getattr(self, "h", None):
            self.n.lease_destroy(self.h)
            self.h = None

    def register(self, w): self.n.lease_register(self.h, w.encode())
    def unregister(self, w): self.n.lease_unregister(self.h, w.encode())
    def is_registered(self, w): return bool(self.n.lease_is_registered(self.h, w.encode()))

    def next(self, w):
        kind, idx = C.c_int(), C.c_uint32()
        off, ln, res, ep = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        st = self.n.lease_next(self.h, w.encode(), C.byref(kind), C.byref(idx), C.byref(off),
                               C.byref(ln), C.byref(res), C.byref(ep))
        if st != 0:
            return (st, None)
        if kind.value == 0:
            return (0, ("shard", idx.value, off.value, ln.value, res.value))
        if kind.value == 1:
            return (0, ("epoch_end", ep.value))
        return (0, ("pending",))

    def report(self, w, p, off): return self.n.lease_report(self.h, w.encode(), p, off)
    def reclaim(self, w): self.n.lease_reclaim(self.h, w.encode())

    def reclaim_at(self, w, pairs):
        ps = (C.c_uint32 * len(pairs))(*[p for p, _ in pairs])
        os_ = (C.c_uint64 * len(pairs))(*[o for _, o in pairs])
        self.n.lease_reclaim_at(self.h, w.encode(), ps, os_, len(pairs))

    def reclaim_missing(self, live): self.n.lease_reclaim_missing(self.h, ",".join(live).encode())

    def meta(self, p):
        off, ln = C.c_uint64(), C.c_uint64()
        self.n.lease_meta(self.h, p, C.byref(off), C.byref(ln))
        return off.value, ln.value

    def worker_shards(self, w):
        ps = (C.c_uint32 * 4096)()
        os_ = (C.c_uint64 * 4096)()
        k = self.n.lease_worker_shards(self.h, w.encode(), ps, os_, 4096)
        return [(ps[i], os_[i]) for i in range(k)]

    def snapshot(self) -> bytes:
        n = self.n.lease_snapshot(self.h, None, 0)
        buf = (C.c_uint8 * n)()
        self.n.lease_snapshot(self.h, buf, n)
        return bytes(buf)

    def restore(self, b: bytes) -> int:
        buf = (C.c_uint8 * len(b)).from_buffer_copy(b)
        return self.n.lease_restore(self.h, buf, len(b))

    def epoch(self): return self.n.lease_epoch(self.h)
    def epochs_completed(self): return self.n.lease_epochs_completed(self.h)
    def cursor(self): return self.n.lease_cursor(self.h)

    def permutation(self):
        n = self.n.lease_permutation(self.h, None, 0)
        out = (C.c_uint32 * max(n, 1))()
        self.n.lease_permutation(self.h, out, n)
        return list(out[:n])

    def reclaimed_count(self): return self.n.lease_reclaimed_count(self.h)
    def in_flight_count(self): return self.n.lease_in_flight_count(self.h)


class Job:
    """The deterministic job protocol (oracle/job_driver.hpp) over or_/ref_ components."""

    def __init__(self, nat: Native, spec: dict, model: int, eta: float, decay: float, B: int,
                 lease_seed: int, partitions: int, ring, per_worker: int = 0, w0=None):
        self.n = nat
        self.dim = spec["dim"]
        w0a = None if w0 is None else np.ascontiguousarray(w0, dtype=np.float64)
        self._w0 = w0a
        self.h = nat.job_create(spec["size"], spec["dim"], spec["seed"], spec.get("noise", 0.0),
                                int(spec.get("sign_labels", False)), model, eta, decay, B,
                                per_worker, lease_seed, partitions, ",".join(ring).encode(),
                                _dp(w0a) if w0a is not None else None)

    def __del__(self):
        if getattr(self, "h", None):
            self.n.job_destroy(self.h)
            self.h = None

    def schedule(self, switch_t: int, out: bool, ids):
        self.n.job_schedule(self.h, switch_t, 1 if out else 0, ",".join(ids).encode())

    def step(self):
        loss, cnt = C.c_double(), C.c_uint64()
        rc = self.n.job_step(self.h, C.byref(loss), C.byref(cnt))
        if rc != 0:
            raise RuntimeError(f"oracle job_step rc={rc}")
        return loss.value, cnt.value

    def params(self) -> np.ndarray:
        w = np.zeros(self.dim, dtype=np.float64)
        self.n.job_params(self.h, _dp(w))
        return w

    def plan(self):
        """[(worker, [(epoch, id), ...]), ...] of the last step, in ring order."""
        out = []
        for r in range(self.n.job_ring_size(self.h)):
            cap = 1 << 20
            ep = (C.c_uint64 * cap)()
            ids = (C.c_uint64 * cap)()
            name = C.create_string_buffer(256)
            n = C.c_size_t()
            self.n.job_plan(self.h, r, name, 256, ep, ids, cap, C.byref(n))
            out.append((name.value.decode(), list(zip(ep[:n.value], ids[:n.value]))))
        return out

    # ---- recovery (job_driver.hpp restore / fail_approximate)
    def snapshot(self) -> "Snapshot":
        """JobCheckpoint at the current mini-batch boundary (params, t, pipeline state)."""
        return Snapshot(self, self.n.job_snapshot(self.h))

    def restore(self, snap: "Snapshot", ring) -> None:
        """Consistent recovery: resume from `snap` with the workers in `ring`."""
        self.n.job_restore(self.h, snap.h, ",".join(ring).encode())

    def fail_approximate(self, failed) -> None:
        """Approximate recovery: redo the last mini-batch without the `failed` workers."""
        self.n.job_fail_approximate(self.h, ",".join(failed).encode())

    def log_text(self) -> str:
        ln = C.c_size_t()
        self.n.job_log_text(self.h, None, 0, C.byref(ln))
        buf = C.create_string_buffer(ln.value + 1)
        self.n.job_log_text(self.h, buf, ln.value + 1, C.byref(ln))
        return buf.value.decode()


class Snapshot:
    def __init__(self, job: Job, h):
        self.job, self.h = job, h

    def __del__(self):
        if getattr(self, "h", None) and getattr(self.job, "h", None):
            self.job.n.job_snap_free(self.job.h, self.h)
            self.h = None


def check_coverage(nat: Native, log_text: str, n: int):
    with tempfile.NamedTemporaryFile("w", suffix=".log", delete=False) as f:
        f.write(log_text)
        path = f.name
    try:
        fe = C.c_uint64()
        detail = C.create_string_buffer(512)
        ok = nat.check_coverage(path.encode(), n, C.byref(fe), detail, 512)
        return bool(ok), fe.value, detail.value.decode()
    finally:
        os.unlink(path)


def replay(nat: Native, log_text: str, model: int, spec: dict, w0, eta, decay, ring_order=True):
    with tempfile.NamedTemporaryFile("w", suffix=".log", delete=False) as f:
        f.write(log_text)
        path = f.name
    try:
        w0a = np.ascontiguousarray(w0, dtype=np.float64)
        w = np.zeros_like(w0a)
        b = C.c_uint64()
        err = C.create_string_buffer(512)
        ok = nat.replay(path.encode(), model, spec["size"], spec["dim"], spec["seed"],
                        spec.get("noise", 0.0), int(spec.get("sign_labels", False)), _dp(w0a),
                        eta, decay, 1 if ring_order else 0, _dp(w), C.byref(b), err, 512)
        return bool(ok), w, b.value, err.value.decode()
    finally:
        os.unlink(path)


def ring_reduce(nat: Native, inputs: np.ndarray, average=False) -> np.ndarray:
    inputs = np.ascontiguousarray(inputs, dtype=np.float64)
    n, ln = inputs.shape
    out = np.zeros(ln, dtype=np.float64)
    nat.ring_reduce(_dp(inputs), n, ln, 1 if average else 0, _dp(out))
    return out
