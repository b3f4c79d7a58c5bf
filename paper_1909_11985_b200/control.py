"""Control plane of one-process-per-GPU jobs: the reference's leader + Fabric messages
(coordination.cpp, transport.hpp:90-100) carried by a torch.distributed
Store (the TCPStore of the job's rendezvous), so the scheduler-facing scale operations work
when every GPU runs its own process.

    scale_out(ranks)   leader only.  The newcomer processes (idle, polling) build their worker
                       -- CUDA context, HBM dataset, buffers, kernels -- while the ring keeps
                       training, then report Ready with their IPC handles.  When all are
                       Ready the leader fixes switch_t = t_cur + max(1, ceil(T_a / T_b))
                       (with a floor that lets every follower see the
                       decision before it is due), publishes it with its host protocol state,
                       and every process schedules the event; at switch_t the ring copies the
                       consolidated model (and momentum) into the newcomers over NVLink.
    scale_in(ranks)    leader only; switch_t = t_cur + k; the leavers' step() answers Exit.
    Retry              while a scaling operation is pending.
    notify_batch_end   every ring process after each step(): the leader checks Ready, the
                       followers pick up decisions (every `poll_every` mini-batches; a
                       decision is due at least `margin` mini-batches after it is made).
    straggler          every ring process publishes its worker's recent mini-batch times;
                       the leader applies the 1.2x-median-for-10 rule.

Keys (under prefix "edl/"): cmd/<n> (JSON: kind, ids, ranks, ring[, switch_t]),
ready/<n>/<rank> (newcomer handle blob), switch/<n> (JSON switch_t + hex host state),
blob/<n>/<rank> (ring process handle blob), times/<rank> (JSON recent step times).
"""
from __future__ import annotations

import json
import math
import time

from . import _lib
from .runtime import Job, switch_delay

K_SLOTS = 4  # csrc/runtime.hpp kSlots: host steps in flight ahead of the device


def wid(rank: int) -> str:
    return f"w{rank:02d}"


class ElasticGroup:
    """One per process.  `ranks_of_ring`: process ranks whose workers form the initial ring
    (worker ids w<rank>); the leader is the lowest rank of the current ring."""

    def __init__(self, store, rank: int, ring_ranks, t_a_ms: float = 500.0, poll_every: int = 8,
                 prefix: str = "edl/"):
        self.store = store
        self.rank = rank
        self.ring_ranks = sorted(ring_ranks)
        self.t_a_ms = t_a_ms
        self.poll_every = max(1, poll_every)
        self.margin = self.poll_every + 2 * K_SLOTS + 2
        self.p = prefix
        self.n_cmd = 0          # next command index this process has not handled yet
        self.pending = None     # leader: scale-out command waiting for Ready
        self.pending_until = -1  # any process: switch_t of the last scheduled event
        self.last_event = None  # (kind, ids, switch_t) of the last event scheduled here

    # ------------------------------------------------------------------ store helpers
    def _k(self, *parts) -> str:
        return self.p + "/".join(str(x) for x in parts)

    def _has(self, key: str) -> bool:
        return self.store.check([self._k(key) if not key.startswith(self.p) else key])

    def _get(self, key: str) -> bytes:
        return self.store.get(key)

    def _set(self, key: str, val) -> None:
        self.store.set(key, val if isinstance(val, (bytes, str)) else json.dumps(val))

    @property
    def leader(self) -> int:
        return self.ring_ranks[0]

    def busy(self, job: Job) -> bool:
        return self.pending is not None or job.t <= self.pending_until

    def _delay(self, job: Job) -> int:
        tb = job.median_step_ms()
        k = switch_delay(self.t_a_ms, tb) if tb > 0 else 1
        return max(k, self.margin)

    # ------------------------------------------------------------------ leader API
    def scale_out(self, job: Job, ranks) -> int:
        """Stop-free scale-out of the processes `ranks`.  Returns -1: the
        switch is fixed once they are Ready (notify_batch_end reports it)."""
        self._check_leader()
        if self.busy(job):
            raise _lib.EdlError(_lib.EDL_RETRY, "a scaling operation is in progress")
        ranks = sorted(ranks)
        cmd = {"kind": "out", "ranks": ranks, "ids": [wid(r) for r in ranks],
               "ring": job.ring(), "ring_ranks": self.ring_ranks}
        self._set(self._k("cmd", self.n_cmd), cmd)
        self.pending = (self.n_cmd, cmd)
        return -1

    def scale_in(self, job: Job, ranks) -> int:
        """Graceful scale-in of the processes `ranks` at t + k."""
        self._check_leader()
        if self.busy(job):
            raise _lib.EdlError(_lib.EDL_RETRY, "a scaling operation is in progress")
        ranks = sorted(ranks)
        if self.leader in ranks:
            raise _lib.EdlError(_lib.EDL_EINVAL, "scale_in of the leader: hand off first")
        switch_t = job.t + self._delay(job)
        ids = [wid(r) for r in ranks]
        self._set(self._k("cmd", self.n_cmd), {"kind": "in", "ranks": ranks, "ids": ids,
                                               "switch_t": switch_t})
        self._apply_in(job, ranks, ids, switch_t)
        self.n_cmd += 1
        return switch_t

    def _check_leader(self):
        if self.rank != self.leader:
            raise _lib.EdlError(_lib.EDL_EINVAL, "scale operations are issued by the leader")

    def _apply_in(self, job, ranks, ids, switch_t):
        job.schedule(switch_t, False, ids)
        self.pending_until = switch_t
        self.last_event = ("in", ids, switch_t)
        self.ring_ranks = [r for r in self.ring_ranks if r not in ranks]

    # ------------------------------------------------------------------ every ring process
    def notify_batch_end(self, job: Job):
        """Call after each job.step() on every ring process.  Returns the (kind, ids,
        switch_t) of an event scheduled by this call, else None."""
        if self.rank == self.leader and self.pending is not None:
            return self._leader_poll_ready(job)
        if self.rank != self.leader and job.t % self.poll_every == 0:
            return self._follower_poll(job)
        return None

    def _leader_poll_ready(self, job: Job):
        n, cmd = self.pending
        keys = [self._k("ready", n, r) for r in cmd["ranks"]]
        if not self.store.check(keys):
            return None
        switch_t = job.t + self._delay(job)
        state = job.export_state()
        self._set(self._k("switch", n), {"switch_t": switch_t, "state": state.hex()})
        self._apply_out(job, n, cmd, switch_t)
        self.pending = None
        self.n_cmd = n + 1
        return ("out", cmd["ids"], switch_t)

    def _apply_out(self, job, n, cmd, switch_t):
        job.schedule(switch_t, True, cmd["ids"], [-1] * len(cmd["ids"]))
        for r in cmd["ranks"]:
            job.import_handles(self._get(self._k("ready", n, r)))
        self._set(self._k("blob", n, self.rank), job.export_handles())
        self.pending_until = switch_t
        self.last_event = ("out", cmd["ids"], switch_t)
        self.ring_ranks = sorted(self.ring_ranks + cmd["ranks"])

    def _follower_poll(self, job: Job):
        ck = self._k("cmd", self.n_cmd)
        if not self.store.check([ck]):
            return None
        cmd = json.loads(self._get(ck))
        if cmd["kind"] == "in":
            if job.t >= cmd["switch_t"]:
                raise _lib.EdlError(_lib.EDL_VERSION_MISMATCH, "scale_in decision arrived late")
            self._apply_in(job, cmd["ranks"], cmd["ids"], cmd["switch_t"])
            self.n_cmd += 1
            return ("in", cmd["ids"], cmd["switch_t"])
        sk = self._k("switch", self.n_cmd)
        if not self.store.check([sk]):
            return None  # newcomers not Ready yet
        sw = json.loads(self._get(sk))
        if job.t >= sw["switch_t"]:
            raise _lib.EdlError(_lib.EDL_VERSION_MISMATCH, "scale_out decision arrived late")
        self._apply_out(job, self.n_cmd, cmd, sw["switch_t"])
        self.n_cmd += 1
        return ("out", cmd["ids"], sw["switch_t"])

    # ------------------------------------------------------------------ newcomer process
    def join(self, cfg, device: int, timeout_s: float = 600.0, poll_s: float = 0.001) -> Job:
        """Idle process: wait for a scale-out command naming this rank, build the newcomer
        (the expensive part, while the ring trains), report Ready, then adopt the leader's
        state and switch_t.  The caller steps the returned job (host-only until switch_t)."""
        t0 = time.time()
        while True:
            ck = self._k("cmd", self.n_cmd)
            if self.store.check([ck]):
                cmd = json.loads(self._get(ck))
                if cmd["kind"] == "out" and self.rank in cmd["ranks"]:
                    break
                if cmd["kind"] == "in":
                    self.ring_ranks = [r for r in self.ring_ranks if r not in cmd["ranks"]]
                elif self.store.check([self._k("switch", self.n_cmd)]):
                    self.ring_ranks = sorted(self.ring_ranks + cmd["ranks"])
                else:
                    time.sleep(poll_s)  # another rank's scale-out, not decided yet
                    continue
                self.n_cmd += 1
                continue
            if time.time() - t0 > timeout_s:
                raise _lib.EdlError(_lib.EDL_TIMEOUT, "no scale-out command for this rank")
            time.sleep(poll_s)
        n = self.n_cmd
        job = Job.joining(cfg, cmd["ring"], cmd["ids"], wid(self.rank), device, self.rank,
                          1 << 62)
        self._set(self._k("ready", n, self.rank), job.export_handles())
        sk = self._k("switch", n)
        self._wait(sk, t0, timeout_s)
        sw = json.loads(self._get(sk))
        job.adopt_state(bytes.fromhex(sw["state"]), sw["switch_t"])
        for r in cmd["ring_ranks"]:
            bk = self._k("blob", n, r)
            self._wait(bk, t0, timeout_s)
            job.import_handles(self._get(bk))
        for r in cmd["ranks"]:
            if r != self.rank:
                job.import_handles(self._get(self._k("ready", n, r)))
        self.ring_ranks = sorted(cmd["ring_ranks"] + cmd["ranks"])
        self.n_cmd = n + 1
        self.pending_until = sw["switch_t"]
        self.last_event = ("out", cmd["ids"], sw["switch_t"])
        return job

    def _wait(self, key: str, t0: float, timeout_s: float, poll_s: float = 0.001) -> None:
        while not self.store.check([key]):
            if time.time() - t0 > timeout_s:
                raise _lib.EdlError(_lib.EDL_TIMEOUT, f"control plane: {key} never arrived")
            time.sleep(poll_s)

    # ------------------------------------------------------------------ stragglers
    def publish_times(self, job: Job, window: int) -> None:
        """Ring process: this worker's last `window` mini-batch device times."""
        self._set(self._k("times", self.rank),
                  {"t": job.t, "ms": job.worker_ms(wid(self.rank))[-window:]})

    def straggler(self, window: int = 10, factor: float = 1.2):
        """Leader: the ring rank whose worker was over factor x the per-mini-batch median in
        each of the last `window` mini-batches, from the published times
        (every ring process must have published), or None."""
        from .runtime import detect_straggler
        rows = []
        for r in self.ring_ranks:
            k = self._k("times", r)
            if not self.store.check([k]):
                return None
            ms = json.loads(self._get(k))["ms"]
            if len(ms) < window:
                return None
            rows.append(ms[-window:])
        dur = [[rows[w][b] for w in range(len(rows))] for b in range(window)]
        i = detect_straggler(dur, window, factor)
        return None if i is None or math.isnan(dur[-1][i]) else self.ring_ranks[i]
