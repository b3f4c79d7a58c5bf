"""Failure recovery (§4.2) on the host protocol (dry-run jobs):
consistent recovery from a checkpoint with the survivors, approximate recovery that redoes
the failed mini-batch, and the no-checkpoint restart.  The assignment logs must equal the
oracle job driver's (oracle/job_driver.hpp restore / fail_approximate) byte for byte, and
pass the reference's coverage audit."""
import os

import pytest

from oracle import api, reference, restated
from paper_1909_11985_b200 import _lib
from paper_1909_11985_b200 import runtime as rt

SPEC = {"size": 2000, "dim": 8, "seed": 1, "noise": 0.0}
RING = ["w00", "w01", "w02"]


def _cfg(**kw):
    base = dict(model=rt.LEAST_SQUARES, size=SPEC["size"], dim=SPEC["dim"], seed=1, noise=0.0,
                eta=0.05, batch=64, lease_seed=7, partitions=16, dry_run=True)
    base.update(kw)
    return rt.JobConfig(**base)


def _steps(job, n):
    for _ in range(n):
        job.step()


@pytest.mark.parametrize("native", [restated, reference])
def test_consistent_recovery_matches_oracle(tmp_path, native):
    nat = native()
    job = rt.Job(_cfg(), RING)
    oj = api.Job(nat, SPEC, 0, 0.05, 0.0, 64, 7, 16, RING)
    _steps(job, 20)
    for _ in range(20):
        oj.step()
    path = str(tmp_path / "ckpt.bin")
    job.save_checkpoint(path)
    snap = oj.snapshot()
    _steps(job, 8)
    for _ in range(8):
        oj.step()
    rep = job.fail(["w01"], approximate=False)
    assert rep["mode"] == "consistent" and rep["status"] == "Ok" and rep["t_resume"] == 20
    oj.restore(snap, ["w00", "w02"])
    assert job.ring() == ["w00", "w02"]
    _steps(job, 40)
    for _ in range(40):
        oj.step()
    assert job.log_text() == oj.log_text()
    ok, _, detail = api.check_coverage(nat, job.log_text(), SPEC["size"])
    assert ok, detail


@pytest.mark.parametrize("native", [restated, reference])
def test_approximate_recovery_redoes_the_minibatch(native):
    nat = native()
    job = rt.Job(_cfg(appx_recovery=True), RING)
    oj = api.Job(nat, SPEC, 0, 0.05, 0.0, 64, 7, 16, RING)
    _steps(job, 25)
    for _ in range(25):
        oj.step()
    rep = job.fail(["w02"], approximate=True)
    assert rep["mode"] == "approximate" and rep["t_resume"] == 24 and rep["version"] == 2
    oj.fail_approximate(["w02"])
    _steps(job, 40)
    for _ in range(40):
        oj.step()
    assert job.log_text() == oj.log_text()
    ok, _, detail = api.check_coverage(nat, job.log_text(), SPEC["size"])
    assert ok, detail


def test_no_checkpoint_restarts_survivors_from_initial_state():
    job = rt.Job(_cfg(), RING)
    _steps(job, 5)
    rep = job.fail(["w00"], approximate=False)
    assert rep["status"] == "NoCheckpoint" and rep["t_resume"] == 0
    assert job.ring() == ["w01", "w02"] and job.t == 0
    _steps(job, 70)
    ok, _, detail = api.check_coverage(restated(), job.log_text(), SPEC["size"])
    assert ok, detail


def test_recovery_errors(tmp_path):
    job = rt.Job(_cfg(), RING)
    _steps(job, 3)
    with pytest.raises(_lib.EdlError) as e:
        job.fail(["w01"], approximate=True)  # boundary state not kept
    assert e.value.code == _lib.EDL_EINVAL
    with pytest.raises(_lib.EdlError) as e:
        job.fail(["w09"])
    assert e.value.code == _lib.EDL_UNKNOWN_WORKER
    with pytest.raises(_lib.EdlError):
        job.fail(RING)  # nobody survives
    path = str(tmp_path / "c.bin")
    job.save_checkpoint(path)
    other = rt.Job(_cfg(batch=32), RING)
    with pytest.raises(_lib.EdlError) as e:
        other.load_checkpoint(path)
    assert e.value.code == _lib.EDL_SHAPE_MISMATCH
    data = open(path, "rb").read()
    with open(path, "wb") as f:
        f.write(data[: len(data) // 2])
    with pytest.raises(_lib.EdlError) as e:
        job.load_checkpoint(path)
    assert e.value.code == _lib.EDL_ETRUNCATED
    with pytest.raises(_lib.EdlError) as e:
        job.load_checkpoint(os.path.join(str(tmp_path), "missing.bin"))
    assert e.value.code == _lib.EDL_EIO
