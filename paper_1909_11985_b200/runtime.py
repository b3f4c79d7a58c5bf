"""Elastic job runtime — Python face of the C ABI (include/edl_b200.h, csrc/runtime.cpp).

Mirrors the reference's (spec-only) job/worker API: scale_out / scale_in / step with
notify_batch_end folded in / split_batch (Table 1).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib

LEAST_SQUARES, LOGISTIC, MLP = 0, 1, 2


def split_batch(B: int, p: int) -> list:
    """SPEC.md:339-347; raises EdlError(Invalid) when B < p."""
    out = (C.c_int64 * max(1, p))()
    _lib.check(_lib.lib().edl_split_batch(B, p, out))
    return list(out[:p])


def switch_delay(t_a_ms: float, t_b_ms: float) -> int:
    """k = max(1, ceil(T_a / T_b))."""
    return _lib.lib().edl_switch_delay(t_a_ms, t_b_ms)


def eta_at(eta: float, decay: float, t: int) -> float:  # trainer.hpp:27-29
    return _lib.lib().edl_eta_at(eta, decay, t)


def detect_straggler(durations, window: int = 10, factor: float = 1.2):
    """durations[batch][worker] (NaN = absent) -> index of the worker slower
    than factor x the per-batch median in each of the last `window` batches, or None."""
    d = np.ascontiguousarray(durations, dtype=np.float64)
    if d.ndim != 2:
        raise ValueError("durations must be [n_batches][n_workers]")
    out = C.c_int32(-1)
    _lib.check(_lib.lib().edl_detect_straggler(
        d.ctypes.data_as(C.POINTER(C.c_double)), d.shape[0], d.shape[1], window, factor,
        C.byref(out)))
    return None if out.value < 0 else out.value


@dataclass
class JobConfig:
    model: int = LEAST_SQUARES
    size: int = 8192
    dim: int = 64
    seed: int = 1
    noise: float = 0.01
    sign_labels: bool = False
    num_classes: int = 4096
    layers: int = 8
    hidden: int = 4096
    eta: float = 0.05
    decay: float = 0.0
    momentum: float = 0.0
    batch: int = 64
    per_worker_batch: int = 0
    lease_seed: int = 7
    partitions: int = 0
    max_workers: int = 1
    init_seed: int = 0
    t_a_ms: float = 500.0
    keep_log: bool = True
    dry_run: bool = False
    appx_recovery: bool = field(
        default_factory=lambda: os.environ.get("USE_APPX_RECOVERY", "0") not in ("", "0"))

    def to_c(self) -> _lib.EdlJobConfig:
        c = _lib.EdlJobConfig()
        c.model = self.model
        c.data = _lib.EdlSyntheticSpec(self.size, self.dim, self.seed, self.noise,
                                       int(self.sign_labels))
        c.num_classes, c.layers, c.hidden = self.num_classes, self.layers, self.hidden
        c.eta, c.decay, c.momentum = self.eta, self.decay, self.momentum
        c.batch, c.per_worker_batch = self.batch, self.per_worker_batch
        c.lease_seed, c.partitions, c.max_workers = self.lease_seed, self.partitions, self.max_workers
        c.init_seed, c.t_a_ms, c.keep_log = self.init_seed, self.t_a_ms, int(self.keep_log)
        c.dry_run = int(self.dry_run)
        c.appx_recovery = int(bool(self.appx_recovery))
        return c


@dataclass
class StepReport:
    t: int
    version: int
    ring_size: int
    switched: bool
    count: int
    loss: float
    step_ms: float
    stall_ms: float

    @staticmethod
    def of(r: _lib.EdlStepReport) -> "StepReport":
        return StepReport(r.t, r.version, r.ring_size, bool(r.switched), r.count, r.loss,
                          r.step_ms, r.stall_ms)


class Job:
    """One elastic data-parallel SGD job (JobState)."""

    def __init__(self, cfg: JobConfig, ring, devices=None):
        self._L = _lib.lib()
        self.cfg = cfg
        ring = list(ring)
        devices = list(devices) if devices is not None else [0] * len(ring)
        h = C.c_void_p()
        c = cfg.to_c()
        dev = (C.c_int32 * len(devices))(*devices)
        _lib.check(self._L.edl_job_create(C.byref(c), _lib.cstrs(ring), dev, len(ring), C.byref(h)))
        self._h = h
        self._devices = dict(zip(ring, devices))  # worker -> GPU (replace_straggler's default)

    @classmethod
    def joining(cls, cfg: JobConfig, ring, newcomers, self_id: str, device: int, rank: int,
                switch_t: int) -> "Job":
        """Scale-out across processes (one process per GPU): this process's newcomer
        `self_id` (one of `newcomers`, each hosted by its own process) on `device` joins the
        job whose current ring is `ring` at `switch_t`.  The ring's processes schedule the
        same event with device -1 (`schedule(switch_t, True, newcomers, [-1] * k)`); handles
        are exchanged before the switch; until then step() replays the lease protocol
        without device work."""
        self = cls.__new__(cls)
        self._L = _lib.lib()
        self.cfg = cfg
        ring = list(ring)
        h = C.c_void_p()
        c = cfg.to_c()
        newcomers = list(newcomers)
        _lib.check(self._L.edl_job_create_joining(C.byref(c), _lib.cstrs(ring), len(ring),
                                                  _lib.cstrs(newcomers), len(newcomers),
                                                  self_id.encode(), device, rank, switch_t,
                                                  C.byref(h)))
        self._h = h
        self._devices = {self_id: device}
        return self

    def close(self):
        if getattr(self, "_h", None):
            self._L.edl_job_destroy(self._h)
            self._h = None

    __del__ = close

    def step(self) -> StepReport:
        r = _lib.EdlStepReport()
        _lib.check(self._L.edl_job_step(self._h, C.byref(r)))
        return StepReport.of(r)

    def sync(self) -> StepReport:
        r = _lib.EdlStepReport()
        _lib.check(self._L.edl_job_sync(self._h, C.byref(r)))
        return StepReport.of(r)

    def scale_out(self, ids, devices=None) -> int:
        """Stop-free scale-out.  Newcomers are prepared on a side thread
        while the job keeps stepping; once they are Ready the switch is set to
        t + max(1, ceil(T_a / T_b)).  Returns -1 (switch pending); the StepReport of the switch
        mini-batch has switched=True.  Raises EdlError(Retry) while another op is pending."""
        ids = list(ids)
        devices = list(devices) if devices is not None else [0] * len(ids)
        st = C.c_int64()
        dev = (C.c_int32 * len(devices))(*devices)
        _lib.check(self._L.edl_job_scale_out(self._h, _lib.cstrs(ids), dev, len(ids), C.byref(st)))
        self._devices.update(zip(ids, devices))
        return st.value

    def scale_in(self, ids, allowance_ms: float = 30000.0) -> int:
        ids = list(ids)
        st = C.c_int64()
        _lib.check(self._L.edl_job_scale_in(self._h, _lib.cstrs(ids), len(ids), allowance_ms,
                                            C.byref(st)))
        return st.value

    def schedule(self, switch_t: int, out: bool, ids, devices=None) -> None:
        ids = list(ids)
        devices = list(devices) if devices is not None else [0] * len(ids)
        self._devices.update(zip(ids, devices))
        dev = (C.c_int32 * max(1, len(devices)))(*devices)
        _lib.check(self._L.edl_job_schedule(self._h, switch_t, 1 if out else 0, _lib.cstrs(ids),
                                            dev, len(ids)))

    def param_count(self) -> int:
        return self._L.edl_job_param_count(self._h)

    def params(self, worker: str) -> np.ndarray:
        n = self.param_count()
        dt = np.float32 if self.cfg.model == MLP else np.float64
        out = np.empty(n, dtype=dt)
        _lib.check(self._L.edl_job_params(self._h, worker.encode(), out.ctypes.data, out.nbytes))
        return out

    def set_params(self, params: np.ndarray) -> None:
        """Checkpoint restore into every replica (MLP: fp32 master; linear: f64 w)."""
        dt = np.float32 if self.cfg.model == MLP else np.float64
        a = np.ascontiguousarray(params, dtype=dt)
        _lib.check(self._L.edl_job_set_params(self._h, a.ctypes.data, a.nbytes))

    @property
    def t(self) -> int:
        return self._L.edl_job_t(self._h)

    def median_step_ms(self) -> float:
        return self._L.edl_job_median_step_ms(self._h)

    def _text(self, fn) -> str:
        n = C.c_size_t()
        fn(self._h, None, 0, C.byref(n))
        buf = C.create_string_buffer(n.value + 1)
        fn(self._h, buf, n.value + 1, C.byref(n))
        return buf.value.decode()

    def log_text(self) -> str:
        return self._text(self._L.edl_job_log)

    def ring(self) -> list:
        s = self._text(self._L.edl_job_ring)
        return s.split(",") if s else []

    def stream_handle(self) -> int:
        """cudaStream_t of the job's kernels (for CUDA-event timing on the right stream)."""
        return self._L.edl_job_stream(self._h) or 0

    def set_profile(self, on: bool) -> None:
        self._L.edl_job_set_profile(self._h, 1 if on else 0)

    def exchange_mode(self) -> int:
        """0 fused collective after the backward, 1/2 per-layer overlap, 3 reduce-scatter
        routed from the wgrad GEMM epilogues, 4 exchange inside the wgrad GEMMs, 5 reduce-
        scatter on the copy engines, 6 split between the two (include/edl_b200.h
        edl_job_exchange_mode)."""
        return int(self._L.edl_job_exchange_mode(self._h))

    def join(self) -> None:
        """Order the job stream after every launched mini-batch's device work (including a
        deferred push collective on the side stream); no host sync (edl_job_join)."""
        _lib.check(self._L.edl_job_join(self._h))

    PHASES = ("gather", "forward", "loss", "backward", "update", "wgrad", "pair")

    def counters(self) -> dict:
        ms = (C.c_double * len(self.PHASES))()
        steps, launches = C.c_uint64(), C.c_uint64()
        self._L.edl_job_counters(self._h, ms, C.byref(steps), C.byref(launches))
        return {"phase_ms": dict(zip(self.PHASES, list(ms))), "steps": steps.value,
                "launches": launches.value}

    def reset_counters(self) -> None:
        self._L.edl_job_reset_counters(self._h)

    def export_handles(self) -> bytes:
        """CUDA IPC handles of this process's replica and workers (multi-process jobs)."""
        n = C.c_size_t()
        _lib.check(self._L.edl_job_export(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * max(1, n.value))()
        _lib.check(self._L.edl_job_export(self._h, buf, n.value, C.byref(n)))
        return bytes(buf[:n.value])

    def import_handles(self, blob: bytes) -> None:
        buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
        _lib.check(self._L.edl_job_import(self._h, buf, len(blob)))

    def export_state(self) -> bytes:
        """Host protocol state at this boundary (leader side of a scheduler-facing
        scale-out across processes; EdlError(Retry) while a scaling op is pending)."""
        n = C.c_size_t()
        _lib.check(self._L.edl_job_export_state(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * max(1, n.value))()
        _lib.check(self._L.edl_job_export_state(self._h, buf, n.value, C.byref(n)))
        return bytes(buf[:n.value])

    def adopt_state(self, blob: bytes, switch_t: int) -> None:
        """Newcomer process (Job.joining, before its first step): continue from the leader's
        boundary state and switch in at switch_t."""
        buf = (C.c_uint8 * max(1, len(blob))).from_buffer_copy(blob or b"\0")
        _lib.check(self._L.edl_job_adopt_state(self._h, buf, len(blob), switch_t))

    def gather_master(self) -> None:
        _lib.check(self._L.edl_job_gather_master(self._h))

    def lease_snapshot(self) -> bytes:
        n = C.c_size_t()
        self._L.edl_job_lease_snapshot(self._h, None, 0, C.byref(n))
        buf = (C.c_uint8 * n.value)()
        self._L.edl_job_lease_snapshot(self._h, buf, n.value, C.byref(n))
        return bytes(buf)

    # ---- straggler mitigation and profiling
    def worker_ms(self, worker: str) -> list:
        """Device time of `worker`'s share of each of the last completed mini-batches."""
        n = C.c_size_t()
        _lib.check(self._L.edl_job_worker_ms(self._h, worker.encode(), None, 0, C.byref(n)))
        buf = (C.c_double * max(1, n.value))()
        _lib.check(self._L.edl_job_worker_ms(self._h, worker.encode(), buf, n.value,
                                             C.byref(n)))
        return list(buf[:n.value])

    def straggler(self, window: int = 10, factor: float = 1.2):
        """Worker over factor x the per-mini-batch median for `window` consecutive mini-batches
        (the leader's detection rule), or None."""
        n = C.c_size_t()
        buf = C.create_string_buffer(256)
        _lib.check(self._L.edl_job_straggler(self._h, window, factor, buf, 256, C.byref(n)))
        return buf.value.decode() or None

    def set_worker_delay(self, worker: str, us: float) -> None:
        """Inject `us` microseconds of extra device time into every mini-batch of `worker`."""
        _lib.check(self._L.edl_job_set_worker_delay(self._h, worker.encode(), float(us)))

    def mitigate_straggler(self, window: int = 10, factor: float = 1.2,
                           allowance_ms: float = 30000.0):
        """Leader action of PAPER.md:418: scale_in the detected straggler (advise-only callers
        use straggler()).  Returns (worker, switch_t) or None."""
        w = self.straggler(window, factor)
        if w is None or len(self.ring()) < 2:
            return None
        return w, self.scale_in([w], allowance_ms)

    def replace_straggler(self, new_id: str, device: int = None, window: int = 10,
                          factor: float = 1.2, allowance_ms: float = 30000.0):
        """Straggler replacement (BASELINE configs[3]): scale_in the detected straggler, keep
        stepping to its switch, then scale_out `new_id` (on `device`, default the straggler's
        GPU) -- two serialised scaling operations (Retry while one is
        pending).  Returns (straggler, scale_in switch_t, scale_out switch_t or -1 = pending
        until the newcomer is Ready) or None when there is no straggler."""
        got = self.mitigate_straggler(window, factor, allowance_ms)
        if got is None:
            return None
        w, st = got
        dev = self._devices.get(w, 0) if device is None else device
        while self.t <= st:
            self.step()
        return w, st, self.scale_out([new_id], [dev])

    def profile(self, min_p: int, max_p: int = None, steps: int = 20) -> list:
        """from the current parallelism (max_p) scale in one worker at a time
        down to min_p, timing `steps` mini-batches per level.  Returns one dict per level:
        parallelism p, samples/s S(p) = t(p) * p, per-GPU throughput t(p) and GPU efficiency
        t(p) / t(p*) with p* = argmax t(p) (PAPER.md:89 footnote)."""
        ring = self.ring()
        max_p = len(ring) if max_p is None else max_p
        if min_p < 1 or min_p > max_p:
            raise _lib.EdlError(_lib.EDL_EINVAL, "profile: min_p > max_p")
        if max_p != len(ring):
            raise _lib.EdlError(_lib.EDL_EINVAL, "profile: the job must run at max_p")
        levels = []
        p = max_p
        while True:
            self.sync()
            reps = []
            for _ in range(steps):
                self.step()
                reps.append(self.sync())
            ms = sorted(r.step_ms for r in reps)[len(reps) // 2]
            count = sorted(r.count for r in reps)[len(reps) // 2]
            thr = 1e3 * count / ms if ms > 0 else 0.0
            levels.append({"p": p, "samples_per_s": thr, "per_gpu": thr / p,
                           "step_ms": ms, "ring": list(self.ring())})
            if p <= min_p:
                break
            st = self.scale_in([self.ring()[-1]])
            while self.t <= st:
                self.step()
            p -= 1
        best = max(lv["per_gpu"] for lv in levels) or 1.0
        for lv in levels:
            lv["efficiency"] = lv["per_gpu"] / best
        return levels

    # ---- failure recovery (§4.2)
    def save_checkpoint(self, path: str) -> None:
        """JobCheckpoint (params, momentum, t_cur, version, B, lease state) to `path`."""
        _lib.check(self._L.edl_job_save_checkpoint(self._h, os.fsencode(path)))

    def load_checkpoint(self, path: str) -> None:
        """Resume from `path` with the job's current workers (consistent recovery)."""
        _lib.check(self._L.edl_job_load_checkpoint(self._h, os.fsencode(path)))

    def fail(self, ids, approximate: bool = None) -> dict:
        """`ids` failed during the last launched mini-batch.  approximate (default:
        JobConfig.appx_recovery): roll back to that mini-batch's start and redo it without
        them; otherwise resume the survivors from the latest checkpoint (status
        "NoCheckpoint": restarted from the initial state)."""
        if approximate is None:
            approximate = self.cfg.appx_recovery
        arr = _lib.cstrs(ids)
        out = _lib.EdlRecovery()
        rc = self._L.edl_job_fail(self._h, arr, len(ids), 1 if approximate else 0,
                                  C.byref(out))
        _lib.check(rc)
        return {"mode": "approximate" if out.mode else "consistent",
                "status": _lib.STATUS_NAMES.get(out.status, out.status),
                "t_resume": out.t_resume, "version": out.version}
