"""Straggler mitigation and profiling on the device:
per-worker mini-batch durations measured with CUDA events, an injected delay on one worker,
detection after exactly `window` slow mini-batches, scale_in of the straggler, and the
scale-in profile of throughput / GPU efficiency per parallelism."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _job(ring):
    from paper_1909_11985_b200 import runtime as rt
    cfg = rt.JobConfig(model=rt.MLP, size=20000, dim=256, seed=3, noise=0.0, num_classes=256,
                       layers=3, hidden=512, eta=0.05, batch=512, lease_seed=5,
                       partitions=64, init_seed=1, keep_log=True)
    return rt.Job(cfg, ring, [0] * len(ring))


def _run(job, n):
    for _ in range(n):
        job.step()
        job.sync()


def test_injected_straggler_detected_after_window_and_removed():
    from oracle import api, restated
    ring = ["w00", "w01", "w02", "w03"]
    job = _job(ring)
    _run(job, 12)
    assert job.straggler() is None
    base = sorted(job.worker_ms("w02")[-10:])[5]
    assert base > 0
    # PAPER.md:529 delays by 1/3 of the mini-batch time; at this tiny size (tens of us per
    # worker) timer and launch jitter can pull a 1.33x worker under the 1.2x rule for one of
    # the 10 mini-batches, so the test delays by 1/2 (the detection rule is unchanged)
    job.set_worker_delay("w02", 1e3 * base / 2)
    _run(job, 9)
    assert job.straggler() is None  # 9 slow mini-batches: not yet
    _run(job, 1)
    assert job.straggler() == "w02"
    w, st = job.mitigate_straggler()
    assert w == "w02"
    while job.t <= st:
        job.step()
    job.sync()
    assert job.ring() == ["w00", "w01", "w03"]
    ok, _, detail = api.check_coverage(restated(), job.log_text(), 20000)
    assert ok, detail


def test_straggler_replaced_with_exactly_once_coverage():
    """BASELINE configs[3]: the detected straggler leaves (scale_in, its shard back in the
    reclaimed queue) and a replacement joins stop-free; every sample of every epoch is still
    drawn exactly once (the reference's check_coverage) and the log replays in the oracle."""
    from oracle import api, restated
    job = _job(["w00", "w01", "w02", "w03"])
    _run(job, 12)
    base = sorted(job.worker_ms("w01")[-10:])[5]
    job.set_worker_delay("w01", 1e3 * base / 2)
    _run(job, 10)
    got = job.replace_straggler("w04")
    assert got is not None and got[0] == "w01"
    assert job.ring() == ["w00", "w02", "w03"]
    import time
    t_end = time.time() + 60  # the newcomer is prepared on a side thread, then switches in
    while time.time() < t_end:
        job.step()
        if job.ring() == ["w00", "w02", "w03", "w04"]:
            break
    job.sync()
    assert job.ring() == ["w00", "w02", "w03", "w04"]
    _run(job, 30)  # past an epoch boundary (20000 samples / 512 per mini-batch)
    assert job.straggler() is None
    ok, _, detail = api.check_coverage(restated(), job.log_text(), 20000)
    assert ok, detail


def test_profile_scales_in_one_worker_per_level():
    job = _job(["w00", "w01", "w02", "w03"])
    _run(job, 3)
    levels = job.profile(min_p=2, steps=6)
    assert [lv["p"] for lv in levels] == [4, 3, 2]
    assert job.ring() == ["w00", "w01"]
    assert max(lv["efficiency"] for lv in levels) == pytest.approx(1.0)
    for lv in levels:
        assert 0 < lv["efficiency"] <= 1.0 + 1e-12
        assert lv["samples_per_s"] == pytest.approx(lv["per_gpu"] * lv["p"])
