"""SPEC AC3 chaos coverage on the host protocol: seeded random schedules that
mix scale-out, scale-in, checkpoints and failures under both recovery modes (consistent:
back to the latest checkpoint with the survivors; approximate: redo the failed mini-batch
without the failed workers) run through the product job (libedl_b200.so, dry-run: the lease /
membership / log protocol without device work) and through the oracle job driver
(oracle/job_driver.hpp over the restated components, and over the reference's own
ShardManager for a third of the seeds).  Every schedule must give a byte-identical
assignment log, and the log must pass the reference's exactly-once coverage audit
(check_coverage, trainer.cpp / SPEC.md:626).
"""
import random

import pytest

from oracle import api, reference, restated
from paper_1909_11985_b200 import _lib
from paper_1909_11985_b200 import runtime as rt

SPEC = {"size": 1500, "dim": 8, "seed": 3, "noise": 0.0}
IDS = [f"w{k:02d}" for k in range(8)]
N_SCHEDULES = 120


def _cfg(appx):
    return rt.JobConfig(model=rt.LEAST_SQUARES, size=SPEC["size"], dim=SPEC["dim"],
                        seed=SPEC["seed"], noise=0.0, eta=0.05, batch=64, lease_seed=5,
                        partitions=16, max_workers=8, dry_run=True, appx_recovery=appx)


def _schedule(seed, tmp_path):
    rng = random.Random(seed)
    appx = seed % 2 == 1  # both recovery modes across the schedules
    nat = reference() if (seed % 3 == 0 and reference() is not None) else restated()
    ring0 = sorted(rng.sample(IDS, rng.randint(1, 3)))
    job = rt.Job(_cfg(appx), ring0)
    oj = api.Job(nat, SPEC, 0, 0.05, 0.0, 64, 5, 16, ring0)
    steps = rng.randint(60, 110)
    pending = []  # (switch_t, seq, out, ids) of scheduled events not yet installed
    snap = None
    ckpt = str(tmp_path / f"c{seed}.bin")
    kinds = {"out": 0, "in": 0, "fail": 0, "ckpt": 0, "rejected": 0}

    def project(extra=None):
        """Membership after every pending event (switch order, ties in scheduling order), or
        None when one of them would empty the ring, remove a non-member or add a member."""
        m = set(job.ring())
        for _, _, out, ids in sorted(pending + ([extra] if extra else []), key=lambda e: e[:2]):
            if out:
                if m & set(ids):
                    return None
                m |= set(ids)
            elif not set(ids) <= m or not m - set(ids):
                return None
            else:
                m -= set(ids)
        return m

    def schedule(st, out, ids):
        ev = (st, len(kinds) + sum(kinds.values()), out, ids)
        if project(ev) is None:  # the product must refuse it, the oracle never sees it
            with pytest.raises(_lib.EdlError) as e:
                job.schedule(st, out, ids)
            assert e.value.code in (_lib.EDL_EINVAL, _lib.EDL_UNKNOWN_WORKER)
            kinds["rejected"] += 1
            return
        job.schedule(st, out, ids)
        oj.schedule(st, out, ids)
        pending.append(ev)
        kinds["out" if out else "in"] += 1

    for _ in range(steps):
        t = job.t  # the next mini-batch (a consistent recovery rewinds it to the checkpoint)
        pending[:] = [e for e in pending if e[0] >= t]  # installed at the start of step e[0]
        ring = sorted(project() or [])
        r = rng.random()
        if r < 0.08 and len(ring) < 6:
            free = [i for i in IDS if i not in ring]
            ids = sorted(rng.sample(free, rng.randint(1, min(2, len(free)))))
            schedule(t + rng.randint(1, 6), True, ids)
        elif r < 0.16 and len(ring) > 1:
            # usually valid; sometimes the whole projected ring (must be refused)
            k = len(ring) if rng.random() < 0.1 else rng.randint(1, len(ring) - 1)
            schedule(t + rng.randint(1, 6), False, sorted(rng.sample(ring, k)))
        elif r < 0.22 and not pending:
            job.save_checkpoint(ckpt)
            snap = oj.snapshot()
            kinds["ckpt"] += 1
        elif r < 0.27 and not pending and len(job.ring()) > 1 and t > 0 and (appx or snap):
            cur = job.ring()
            failed = sorted(rng.sample(cur, rng.randint(1, len(cur) - 1)))
            survivors = [i for i in cur if i not in failed]
            rep = job.fail(failed, approximate=appx)
            if appx:
                oj.fail_approximate(failed)
            else:
                assert rep["status"] == "Ok"
                oj.restore(snap, survivors)
            assert job.ring() == survivors
            kinds["fail"] += 1
        job.step()
        oj.step()
    text = job.log_text()
    assert text == oj.log_text(), (seed, kinds)
    ok, full_epochs, detail = api.check_coverage(nat, text, SPEC["size"])
    assert ok, (seed, kinds, detail)
    return kinds


def test_chaos_schedules_match_oracle_and_cover_exactly_once(tmp_path):
    total = {"out": 0, "in": 0, "fail": 0, "ckpt": 0, "rejected": 0}
    for seed in range(N_SCHEDULES):
        for k, v in _schedule(seed, tmp_path).items():
            total[k] += v
    # the schedules really mix every kind of event
    assert all(total[k] >= N_SCHEDULES // 2 for k in ("out", "in", "fail", "ckpt")), total
    assert total["rejected"] > 0, total


def test_fail_while_scaling_is_retry(tmp_path):
    job = rt.Job(_cfg(True), ["w00", "w01"])
    job.step()
    job.schedule(3, True, ["w02"])
    with pytest.raises(_lib.EdlError) as e:
        job.fail(["w01"], approximate=True)
    assert e.value.code == _lib.EDL_RETRY
