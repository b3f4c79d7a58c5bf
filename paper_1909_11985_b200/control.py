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


class SystemClock:
    def now(self) -> float:
        return time.monotonic()


class ManualClock:
    """Injectable clock for deterministic expiry tests (the reference's ManualClock)."""

    def __init__(self, t: float = 0.0):
        self.t = t

    def now(self) -> float:
        return self.t

    def advance(self, dt: float) -> None:
        self.t += dt


class LeaderLease:
    """Lease-backed leader election with compare-and-swap semantics (the reference's
    LeaseStore, coordination.hpp / coordination.cpp:26-117) on a
    torch.distributed Store: the record "address|deadline|generation" of key `job` is
    claimed by an atomic compare_set when it is absent, erased or expired; refresh extends
    the holder's deadline, erase removes it (graceful exit), get reads it.  watch()/poll()
    deliver Elected(address, generation) after each successful claim and Expired within one
    poll after a record expires or is erased.  TTL default 3 s (refresh ttl/3, poll ttl/10).
    Times come from `clock` (monotonic; processes on one node share it)."""

    WON, LOST = "Won", "Lost"
    OK, NOT_LEADER = "Ok", "NotLeader"

    def __init__(self, store, clock=None, ttl: float = 3.0, prefix: str = "edl/leader/"):
        self.store = store
        self.clock = clock or SystemClock()
        self.ttl = ttl
        self.p = prefix
        self._watch = {}   # id -> (job, fn)
        self._seen = {}    # job -> (present, generation) last delivered to watchers
        self._next = 0

    def _key(self, job: str) -> str:
        return self.p + job

    def _read(self, job: str) -> str:
        k = self._key(job)
        return self.store.get(k).decode() if self.store.check([k]) else ""

    @staticmethod
    def _parse(rec: str):
        if not rec or rec.startswith("-"):  # absent, or erased ("-<generation>")
            return None
        addr, dl, gen = rec.rsplit("|", 2)
        return addr, float(dl), int(gen)

    @staticmethod
    def _last_gen(rec: str) -> int:
        if not rec:
            return 0
        if rec.startswith("-"):
            return int(rec[1:])
        return int(rec.rsplit("|", 1)[1])

    def cas_put_if_absent_or_expired(self, job: str, address: str, ttl: float = None):
        """(Won, generation, address) or (Lost, generation, winner's address)."""
        t = self.ttl if ttl is None else ttl
        while True:
            cur = self._read(job)
            rec = self._parse(cur)
            now = self.clock.now()
            if rec is not None and now <= rec[1]:
                return (self.LOST, rec[2], rec[0])
            gen = self._last_gen(cur) + 1
            new = f"{address}|{now + t!r}|{gen}"
            got = self.store.compare_set(self._key(job), cur, new).decode()
            if got == new:
                self.poll()
                return (self.WON, gen, address)
            # somebody changed the record between the read and the swap: look again

    def refresh(self, job: str, address: str, ttl: float = None) -> str:
        t = self.ttl if ttl is None else ttl
        cur = self._read(job)
        rec = self._parse(cur)
        now = self.clock.now()
        if rec is None or rec[0] != address or now > rec[1]:
            return self.NOT_LEADER
        new = f"{address}|{now + t!r}|{rec[2]}"
        return self.OK if self.store.compare_set(self._key(job), cur, new).decode() == new \
            else self.NOT_LEADER

    def erase(self, job: str, address: str) -> str:
        cur = self._read(job)
        rec = self._parse(cur)
        if rec is None or rec[0] != address:
            return self.NOT_LEADER
        new = f"-{rec[2]}"  # keeps the generation counter monotonic across erases
        ok = self.store.compare_set(self._key(job), cur, new).decode() == new
        if ok:
            self.poll()
        return self.OK if ok else self.NOT_LEADER

    def get(self, job: str):
        """(address, deadline, generation) of the unexpired record, or None."""
        rec = self._parse(self._read(job))
        return rec if rec is not None and self.clock.now() <= rec[1] else None

    def watch(self, job: str, fn) -> int:
        self._next += 1
        self._watch[self._next] = (job, fn)
        self._seen.setdefault(job, (False, 0))
        return self._next

    def unwatch(self, wid_: int) -> None:
        self._watch.pop(wid_, None)

    def poll(self) -> None:
        """Deliver Elected / Expired to the watchers of every watched job (call every
        ttl/10, or after own claims / erases)."""
        for job in {j for j, _ in self._watch.values()}:
            rec = self.get(job)
            was_present, was_gen = self._seen.get(job, (False, 0))
            evs = []
            if rec is not None and rec[2] != was_gen:
                if was_present:
                    evs.append(("Expired", job, "", 0))
                evs.append(("Elected", job, rec[0], rec[2]))
                self._seen[job] = (True, rec[2])
            elif rec is None and was_present:
                evs.append(("Expired", job, "", 0))
                self._seen[job] = (False, was_gen)
            for ev in evs:
                for j, fn in list(self._watch.values()):
                    if j == job:
                        fn(ev)


def wid(rank: int) -> str:
    return f"w{rank:02d}"


class ElasticGroup:
    """One per process.  `ring_ranks`: process ranks whose workers form the initial ring
    (worker ids w<rank>).  The leader is the holder of `lease` (LeaderLease) when one is
    given, else the lowest rank of the current ring."""

    def __init__(self, store, rank: int, ring_ranks, t_a_ms: float = 500.0, poll_every: int = 8,
                 prefix: str = "edl/", lease: "LeaderLease" = None, job_key: str = "job"):
        self.store = store
        self.rank = rank
        self.ring_ranks = sorted(ring_ranks)
        # leader election: with a LeaderLease the leader is whoever holds the
        # job's lease record (address "rank:<r>"); without one, the lowest ring rank
        self.lease = lease
        self.job_key = job_key
        self._leader_rank = None
        self._refreshed = 0.0
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

    def _get(self, key: str) -> bytes:
        return self.store.get(key)

    def _set(self, key: str, val) -> None:
        self.store.set(key, val if isinstance(val, (bytes, str)) else json.dumps(val))

    @property
    def leader(self) -> int:
        if self.lease is None:
            return self.ring_ranks[0]
        if self._leader_rank is None:
            rec = self.lease.get(self.job_key)
            self._leader_rank = int(rec[0].split(":")[1]) if rec else -1
        return self._leader_rank

    def elect(self) -> bool:
        """Ring process: try to become the leader (cas_put_if_absent_or_expired)."""
        st, gen, addr = self.lease.cas_put_if_absent_or_expired(self.job_key, f"rank:{self.rank}")
        self._leader_rank = int(addr.split(":")[1])
        self._refreshed = self.lease.clock.now()
        self.generation = gen
        return st == LeaderLease.WON

    def leave(self, job: Job) -> None:
        """A leaving leader's graceful exit: erase the coordination record so the
        survivors elect a successor at once; the job meta-data (t_cur, B, pipeline cursor) is
        already identical in every process (each replays the leader's decisions)."""
        if self.lease is not None and self.leader == self.rank:
            self.lease.erase(self.job_key, f"rank:{self.rank}")
            self._leader_rank = None

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
        if self.leader in ranks and self.lease is None:
            raise _lib.EdlError(_lib.EDL_EINVAL, "scale_in of the leader needs leader election")
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
        if self.lease is not None:
            if self.leader == self.rank:  # keep the lease: refresh every ttl / 3
                now = self.lease.clock.now()
                if now - self._refreshed > self.lease.ttl / 3:
                    if self.lease.refresh(self.job_key, f"rank:{self.rank}") != LeaderLease.OK:
                        self._leader_rank = None  # lost it (expired and re-elected)
                    self._refreshed = now
            elif job.t % self.poll_every == 0 and job.t > self.pending_until:
                # the leader left (erased) or died (expired): elect a successor
                self._leader_rank = None
                if self.leader < 0 or self.leader not in self.ring_ranks:
                    self.elect()
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
