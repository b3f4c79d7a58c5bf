"""N>1 host path on CPU: two processes (gloo, world_size 2) each host one worker of a
2-member ring in dry-run mode (host protocol only), replay the lease protocol for the whole
ring, exchange their handle blobs and must agree with each other and with the oracle on every
mini-batch's composition, membership and the exactly-once coverage.  The device data path of
the same jobs is covered by tests/test_job_gpu.py and bench.py --gpus N."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SPEC = {"size": 5000, "dim": 8, "seed": 3, "noise": 0.0, "sign_labels": False}
EVENTS = [(7, True, ["w02"]), (15, False, ["w00"]), (22, True, ["w05"])]
STEPS = 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_11985_b200 import runtime as rt
    cfg = rt.JobConfig(model=rt.LEAST_SQUARES, size=SPEC["size"], dim=SPEC["dim"],
                       seed=SPEC["seed"], noise=0.0, batch=96, lease_seed=11, partitions=64,
                       dry_run=True)
    ring = ["w00", "w01"]
    job = rt.Job(cfg, ring, [0 if i == rank else -1 for i in range(len(ring))])
    blob = job.export_handles()
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    for t, o, ids in EVENTS:
        job.schedule(t, o, ids, [0] * len(ids))
    counts = [job.step().count for _ in range(STEPS)]
    logs = [None] * world
    dist.all_gather_object(logs, (job.log_text(), counts, job.ring()))
    if rank == 0:
        out.put(logs)
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_replicated_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    logs = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (log0, c0, ring0), (log1, c1, ring1) = logs
    assert log0 == log1 and c0 == c1 and ring0 == ring1 == ["w01", "w02", "w05"]

    from oracle import api, restated
    oj = api.Job(restated(), SPEC, 2, 0.0, 0.0, 96, 11, 64, ["w00", "w01"])
    for t, o, ids in EVENTS:
        oj.schedule(t, o, ids)
    ocounts = [oj.step()[1] for _ in range(STEPS)]
    assert log0 == oj.log_text()
    assert c0 == ocounts
    ok, fe, detail = api.check_coverage(restated(), log0, SPEC["size"])
    assert ok, detail


def _worker_static(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1909_11985_b200 import runtime as rt
    # bench.py's N-GPU shape: one member per process, fixed per-worker batch
    cfg = rt.JobConfig(model=rt.MLP, size=1 << 16, dim=64, seed=1, noise=0.0, num_classes=64,
                       layers=2, hidden=64, batch=512, per_worker_batch=512, lease_seed=7,
                       partitions=0, max_workers=world, init_seed=0, dry_run=True)
    ring = [f"w{r:02d}" for r in range(world)]
    job = rt.Job(cfg, ring, [0 if i == rank else -1 for i in range(world)])
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    counts = [job.step().count for _ in range(STEPS)]
    logs = [None] * world
    dist.all_gather_object(logs, (job.log_text(), counts))
    if rank == 0:
        out.put(logs)
    dist.barrier()
    dist.destroy_process_group()


def test_eight_process_static_ring_protocol():
    """The driver's 8-GPU scaling run: eight processes, one ring member each, replay the same
    lease protocol (every mini-batch 8 x 512 samples) and agree with the oracle."""
    world = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_static, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    logs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(lg == logs[0] for lg in logs)
    log0, c0 = logs[0]
    assert c0 == [8 * 512] * STEPS

    from oracle import api, restated
    spec = {"size": 1 << 16, "dim": 64, "seed": 1, "noise": 0.0, "sign_labels": False}
    ring = [f"w{r:02d}" for r in range(world)]
    oj = api.Job(restated(), spec, 2, 0.0, 0.0, 512 * world, 7, 64, ring, per_worker=512)
    for _ in range(STEPS):
        oj.step()
    assert log0 == oj.log_text()
