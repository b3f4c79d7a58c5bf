"""Worker script for tests/test_multigpu_gpu.py (run under torch.distributed.run, one process
per GPU).  Each rank hosts one ring member; the gradient exchange is the fused NVLink
peer-memory kernel.  Rank 0 checks the results against the CPU oracle and exits non-zero on
a mismatch."""
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


def connect(job, world, rank):
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    dist.barrier()


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ring = [f"w{r:02d}" for r in range(world)]
    devices = [local if r == rank else -1 for r in range(world)]
    failures = []

    # 1. least squares, static ring: f64 ring-order allreduce -> bit-exact vs the oracle
    spec = {"size": 8192, "dim": 64, "seed": 1, "noise": 0.01, "sign_labels": False}
    cfg = rt.JobConfig(model=rt.LEAST_SQUARES, size=spec["size"], dim=spec["dim"], seed=1,
                       noise=0.01, eta=0.05, batch=64 * world, lease_seed=7, partitions=64)
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    reps = []
    for _ in range(60):
        job.step()
        reps.append(job.sync())
    w = job.params(ring[rank])
    oj = api.Job(restated(), spec, 0, 0.05, 0.0, 64 * world, 7, 64, ring)
    ref = [oj.step() for _ in range(60)]
    wref = oj.params()
    if not np.array_equal(w.view(np.uint64), wref.view(np.uint64)):
        failures.append(f"rank {rank}: linear params differ (max {np.abs(w - wref).max()})")
    for rep, (loss, cnt) in zip(reps, ref):
        if rep.count != cnt or float(rep.loss).hex() != float(loss).hex():
            failures.append(f"rank {rank}: linear t={rep.t} loss {rep.loss} vs {loss}")
            break
    if job.log_text() != oj.log_text():
        failures.append(f"rank {rank}: assignment log differs")
    job.close()

    # 2. small MLP: sharded fp32 master + all-gather of bf16 weights over NVLink
    dim, hidden, classes, layers, B, steps = 64, 128, 64, 3, 96, 8
    mspec = {"size": 3000, "dim": dim, "seed": 5}
    cfg = rt.JobConfig(model=rt.MLP, size=3000, dim=dim, seed=5, noise=0.0, num_classes=classes,
                       layers=layers, hidden=hidden, eta=0.1, decay=0.01, batch=B,
                       lease_seed=11, partitions=64, init_seed=3)
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    got = []
    for _ in range(steps):
        job.step()
        got.append(job.sync())
    job.gather_master()
    wm = job.params(ring[rank])
    pj = api.Job(restated(), mspec, 2, 0.0, 0.0, B, 11, 64, ring)
    orc = MLPOracle(dim, hidden, classes, layers, 5, 3, 0.1, 0.01)
    for t in range(steps):
        pj.step()
        plan = [(wk, [i for _, i in s]) for wk, s in pj.plan()]
        ref_loss = orc.step(plan, t)
        if abs(got[t].loss - ref_loss) > 1e-3 * abs(ref_loss):
            failures.append(f"rank {rank}: mlp t={t} loss {got[t].loss} vs {ref_loss}")
    ref = orc.flat_master()
    if np.abs(wm - ref).max() > 1e-3 * np.abs(ref).max() or \
            np.linalg.norm(wm - ref) > 1e-3 * np.linalg.norm(ref):
        failures.append(f"rank {rank}: mlp params max err {np.abs(wm - ref).max()}")
    job.close()

    # 3. an MLP whose layers split into per-GPU row blocks: with the default EDL_OVERLAP the
    #    reduce-scatter rides in the weight-gradient GEMM epilogues (TMA stores into the
    #    owner's receive buffer over NVLink), then per-layer shard update + all-gather
    # (1024-wide layers: whole 256-row tiles per owner at 4 GPUs, so EDL_OVERLAP=4 applies)
    dim, hidden, classes, layers, steps = 256, 1024, 1024, 3, 6
    B = 64 * world
    mspec = {"size": 4000, "dim": dim, "seed": 9}
    cfg = rt.JobConfig(model=rt.MLP, size=4000, dim=dim, seed=9, noise=0.0, num_classes=classes,
                       layers=layers, hidden=hidden, eta=0.1, decay=0.0, batch=B,
                       lease_seed=13, partitions=64, init_seed=4)
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    got = []
    for _ in range(steps):
        job.step()
        got.append(job.sync())
    job.gather_master()
    wm = job.params(ring[rank])
    pj = api.Job(restated(), mspec, 2, 0.0, 0.0, B, 13, 64, ring)
    orc = MLPOracle(dim, hidden, classes, layers, 9, 4, 0.1, 0.0)
    for t in range(steps):
        pj.step()
        plan = [(wk, [i for _, i in s]) for wk, s in pj.plan()]
        ref_loss = orc.step(plan, t)
        if abs(got[t].loss - ref_loss) > 1e-3 * abs(ref_loss):
            failures.append(f"rank {rank}: mlp-rs t={t} loss {got[t].loss} vs {ref_loss}")
    ref = orc.flat_master()
    err = np.abs(wm - ref)
    if err.max() > 2 ** -8 * np.abs(ref).max() or err.mean() > 1e-4 * np.abs(ref).max() \
            or np.linalg.norm(err) > 1e-3 * np.linalg.norm(ref):
        failures.append(f"rank {rank}: mlp-rs params max err {err.max()} mean {err.mean()}")
    job.close()

    # 4. the same job pipelined: no host sync between mini-batches, so with the deferred
    #    all-gather (default) every push collective overlaps the next mini-batch's forward,
    #    whose GEMMs wait on the per-layer weight flags.  Same parameters as section 3.
    job = rt.Job(cfg, ring, devices)
    connect(job, world, rank)
    for _ in range(steps):
        job.step()
    last = job.sync()
    job.gather_master()
    wp = job.params(ring[rank])
    if abs(last.loss - got[-1].loss) > 1e-6 * abs(got[-1].loss):
        failures.append(f"rank {rank}: pipelined last loss {last.loss} vs {got[-1].loss}")
    err = np.abs(wp - ref)
    if err.max() > 2 ** -8 * np.abs(ref).max() or err.mean() > 1e-4 * np.abs(ref).max() \
            or np.linalg.norm(err) > 1e-3 * np.linalg.norm(ref):
        failures.append(f"rank {rank}: pipelined params max err {err.max()} mean {err.mean()}")
    if not np.array_equal(wp, wm):
        failures.append(f"rank {rank}: pipelined params differ from the synced run "
                        f"(max {np.abs(wp - wm).max()})")
    job.close()

    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.barrier()
    dist.destroy_process_group()
    flat = [f for fs in allf for f in fs]
    if rank == 0:
        print("MP-PARITY", "OK" if not flat else "FAIL", flat, flush=True)
    sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
