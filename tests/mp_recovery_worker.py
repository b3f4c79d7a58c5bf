"""Worker script for tests/test_multigpu_gpu.py::test_multi_process_consistent_recovery (run
under torch.distributed.run, one process per GPU, one ring member per process).

Consistent failure recovery across processes (§4.2): every ring
process takes the checkpoint at t=C (a collective: the sharded fp32 master and momentum are
all-gathered, each process writes the same JobCheckpoint); after mini-batch X-1 the last
rank's process dies (it frees its job and stops taking part); the survivors call
fail([its worker]) -- they drop its replica from the collective without touching its memory,
reload the checkpoint (leases as checkpointed, its in-flight shards reclaimed, the ring
re-formed) and go on from t=C.  Checked against the oracle driver's snapshot / restore on the
same schedule: the least-squares job bit-exact (losses, parameters, assignment log), the MLP
(momentum 0.9) within 1e-3 relative.
"""
import os
import sys
import tempfile

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import api, restated  # noqa: E402
from oracle.mlp import MLPOracle  # noqa: E402
from paper_1909_11985_b200 import runtime as rt  # noqa: E402

C, X, END = 5, 9, 16


def connect(job, world, rank):
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    dist.barrier()


def run_case(cfg, spec, model, ring, rank, world, local, tmp, failures, tag):
    devices = [local if r == rank else -1 for r in range(world)]
    dead = ring[-1]
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    got = {}
    path = os.path.join(tmp, f"{tag}_ckpt_r{rank}.bin")
    for _ in range(X):
        rep = job.step()
        got[rep.t] = job.sync()
        if job.t == C:
            job.save_checkpoint(path)  # collective: every ring process, same boundary
    dist.barrier()  # every process finished mini-batch X-1: the failure is between batches
    if ring[rank] == dead:
        job.close()  # the process dies: its device memory is gone
        dist.barrier()  # (test bookkeeping only) the survivors have recovered and finished
        return None
    rec = job.fail([dead], approximate=False)
    if rec["mode"] != "consistent" or rec["status"] != "Ok" or rec["t_resume"] != C:
        failures.append(f"{tag} rank {rank}: recovery {rec}")
    survivors = [w for w in ring if w != dead]
    if job.ring() != survivors:
        failures.append(f"{tag} rank {rank}: ring {job.ring()}")
    while job.t < END:
        rep = job.step()
        got[rep.t] = job.sync()
    # oracle: the same checkpoint / failure schedule
    oj = api.Job(restated(), spec, model if model != rt.MLP else 2, cfg.eta, cfg.decay,
                 cfg.batch, cfg.lease_seed, cfg.partitions, ring)
    orc = MLPOracle(cfg.dim, cfg.hidden, cfg.num_classes, cfg.layers, cfg.seed, cfg.init_seed,
                    cfg.eta, cfg.decay, momentum=cfg.momentum) if model == rt.MLP else None
    ref, snap, osnap = {}, None, None
    t = 0
    while t < X:
        loss, cnt = oj.step()
        if orc is not None:
            loss = orc.step([(wk, [i for _, i in s]) for wk, s in oj.plan()], t)
        ref[t] = loss
        t += 1
        if t == C:
            snap = oj.snapshot()
            if orc is not None:
                osnap = (orc.flat_master().copy(), orc.flat_mom().copy())
    oj.restore(snap, survivors)
    if orc is not None:
        orc.set_state(*osnap)
    for t in range(C, END):
        loss, cnt = oj.step()
        if orc is not None:
            loss = orc.step([(wk, [i for _, i in s]) for wk, s in oj.plan()], t)
        ref[t] = loss
    for t in range(END):
        g_, r_ = got[t].loss, ref[t]
        ok = (float(g_).hex() == float(r_).hex()) if model != rt.MLP else \
            abs(g_ - r_) <= 1e-3 * abs(r_)
        if not ok:
            failures.append(f"{tag} rank {rank}: t={t} loss {g_} vs {r_}")
            break
    if job.log_text() != oj.log_text():
        failures.append(f"{tag} rank {rank}: assignment log differs from the oracle's")
    if model == rt.MLP:
        job.gather_master()
        w = job.params(ring[rank])
        rw = orc.flat_master()
        rel = float(np.linalg.norm(w - rw) / np.linalg.norm(rw))
        if rel > 1e-3:
            failures.append(f"{tag} rank {rank}: params rel L2 {rel}")
    else:
        if not np.array_equal(job.params(ring[rank]).view(np.uint64), oj.params().view(np.uint64)):
            failures.append(f"{tag} rank {rank}: linear params differ")
    dist.barrier()
    return job


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ring = [f"w{r:02d}" for r in range(world)]
    failures, jobs = [], []
    tmp = tempfile.mkdtemp(prefix=f"edl_rec_{rank}_")
    spec = {"size": 8192, "dim": 64, "seed": 1, "noise": 0.01, "sign_labels": False}
    cfg = rt.JobConfig(model=rt.LEAST_SQUARES, size=8192, dim=64, seed=1, noise=0.01, eta=0.05,
                       batch=64 * world, lease_seed=7, partitions=64)
    jobs.append(run_case(cfg, spec, rt.LEAST_SQUARES, ring, rank, world, local, tmp, failures,
                         "linear"))
    mspec = {"size": 4000, "dim": 256, "seed": 9}
    mcfg = rt.JobConfig(model=rt.MLP, size=4000, dim=256, seed=9, noise=0.0, num_classes=1024,
                        layers=3, hidden=1024, eta=0.01, decay=0.0, momentum=0.9,
                        batch=64 * world, lease_seed=13, partitions=64, init_seed=4)
    jobs.append(run_case(mcfg, mspec, rt.MLP, ring, rank, world, local, tmp, failures, "mlp"))
    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.barrier()
    for j in jobs:
        if j is not None:
            j.close()
    dist.barrier()
    dist.destroy_process_group()
    flat = [f for fs in allf for f in fs]
    if rank == 0:
        print("MP-RECOVERY", "OK" if not flat else "FAIL", flat, flush=True)
    sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
