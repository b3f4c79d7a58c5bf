"""Worker script for tests/test_multigpu_gpu.py::test_multi_process_scale_in (run under
torch.distributed.run, one process per GPU, one ring member per process).

Scale-in across processes: every process schedules the same event; at the
switch the fp32 master shards are consolidated into every replica, the leavers' leases are
reclaimed (datapipeline.cpp:73-84), the leavers' processes get notify_batch_end = Exit and stop,
and the survivors continue on the smaller ring with no restart.  Checked against the CPU
oracle driving the same event: the assignment log (bit-exact), the linear job's parameters
(bit-exact f64) and the MLP's loss trajectory / parameters (tolerances of the static tests).
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import api, restated  # noqa: E402
from oracle.mlp import MLPOracle  # noqa: E402
from paper_1909_11985_b200 import runtime as rt  # noqa: E402

SWITCH = 4


def connect(job, world, rank):
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    dist.barrier()


def run(job, ring, rank, steps):
    """Steps until this process's member leaves; returns the synced reports."""
    got = []
    for _ in range(steps):
        rep = job.step()
        if ring[rank] not in job.ring():
            assert rep.switched == 1 and rep.count == 0
            break
        got.append(job.sync())
    return got


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ring = [f"w{r:02d}" for r in range(world)]
    devices = [local if r == rank else -1 for r in range(world)]
    leavers = ring[world // 2:]
    failures = []
    jobs = []

    # 1. least squares: f64 ring-order reduction, bit-exact vs the oracle through the event
    spec = {"size": 8192, "dim": 64, "seed": 1, "noise": 0.01, "sign_labels": False}
    cfg = rt.JobConfig(model=rt.LEAST_SQUARES, size=spec["size"], dim=spec["dim"], seed=1,
                       noise=0.01, eta=0.05, batch=64 * world, lease_seed=7, partitions=64)
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    job.schedule(SWITCH, False, leavers)
    steps = 12
    got = run(job, ring, rank, steps)
    oj = api.Job(restated(), spec, 0, 0.05, 0.0, 64 * world, 7, 64, ring)
    oj.schedule(SWITCH, False, leavers)
    ref = [oj.step() for _ in range(steps)]
    for rep, (loss, cnt) in zip(got, ref):
        if rep.count != cnt or float(rep.loss).hex() != float(loss).hex():
            failures.append(f"rank {rank}: linear t={rep.t} loss {rep.loss} vs {loss}")
            break
    if ring[rank] in leavers:
        if len(got) != SWITCH:
            failures.append(f"rank {rank}: leaver stepped {len(got)} mini-batches")
    else:
        if len(got) != steps:
            failures.append(f"rank {rank}: survivor stepped {len(got)} mini-batches")
        w = job.params(ring[rank])
        if not np.array_equal(w.view(np.uint64), oj.params().view(np.uint64)):
            failures.append(f"rank {rank}: linear params differ after scale-in")
        if job.log_text() != oj.log_text():
            failures.append(f"rank {rank}: linear assignment log differs")
        if job.ring() != ring[:world // 2]:
            failures.append(f"rank {rank}: ring {job.ring()}")
    jobs.append(job)

    # 2. MLP whose layers split into per-GPU row blocks (the default exchange: reduce-scatter
    #    in the wgrad GEMM epilogues + push collective), re-sharded at the switch
    dim, hidden, classes, layers, steps = 256, 1024, 1024, 3, 10
    B = 64 * world
    mspec = {"size": 4000, "dim": dim, "seed": 9}
    cfg = rt.JobConfig(model=rt.MLP, size=4000, dim=dim, seed=9, noise=0.0, num_classes=classes,
                       layers=layers, hidden=hidden, eta=0.1, decay=0.0, batch=B,
                       lease_seed=13, partitions=64, init_seed=4)
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    job.schedule(SWITCH, False, leavers)
    got = run(job, ring, rank, steps)
    pj = api.Job(restated(), mspec, 2, 0.0, 0.0, B, 13, 64, ring)
    pj.schedule(SWITCH, False, leavers)
    orc = MLPOracle(dim, hidden, classes, layers, 9, 4, 0.1, 0.0)
    for t in range(steps):
        pj.step()
        plan = [(wk, [i for _, i in s]) for wk, s in pj.plan()]
        ref_loss = orc.step(plan, t)
        if t < len(got) and abs(got[t].loss - ref_loss) > 1e-3 * abs(ref_loss):
            failures.append(f"rank {rank}: mlp t={t} loss {got[t].loss} vs {ref_loss}")
    if ring[rank] not in leavers:
        job.gather_master()
        wm = job.params(ring[rank])
        ref = orc.flat_master()
        err = np.abs(wm - ref)
        if err.max() > 2 ** -8 * np.abs(ref).max() or err.mean() > 1e-4 * np.abs(ref).max() \
            or np.linalg.norm(err) > 1e-3 * np.linalg.norm(ref):
            failures.append(f"rank {rank}: mlp params max err {err.max()} mean {err.mean()}")
        if job.log_text() != pj.log_text():
            failures.append(f"rank {rank}: mlp assignment log differs")
    jobs.append(job)

    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.barrier()  # the survivors are done with every peer mapping before anyone frees
    for j in jobs:
        j.close()
    dist.barrier()
    dist.destroy_process_group()
    flat = [f for fs in allf for f in fs]
    if rank == 0:
        print("MP-SCALE-IN", "OK" if not flat else "FAIL", flat, flush=True)
    sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
