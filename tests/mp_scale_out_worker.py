"""Worker script for tests/test_multigpu_gpu.py::test_multi_process_scale_out (run under
torch.distributed.run, one process per GPU, one ring member per process).

Stop-free scale-out across processes: the lower half of the ranks start the
job; each upper-half rank builds its newcomer (CUDA context, HBM dataset, buffers) with
`Job.joining` while the ring trains, exchanges handles, replays the lease protocol without
device work, and switches in at t=SWITCH, where the ring's processes copy the consolidated
model into it over NVLink.  Checked against the CPU oracle driving the same event: identical
assignment log, loss trajectory and final parameters within the static tests' tolerances.
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


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    full = [f"w{r:02d}" for r in range(world)]
    half = world // 2
    ring0, newcomers = full[:half], full[half:]
    failures = []

    dim, hidden, classes, layers, steps = 256, 1024, 1024, 3, 10
    B = 64 * world
    mspec = {"size": 4000, "dim": dim, "seed": 9}
    cfg = rt.JobConfig(model=rt.MLP, size=4000, dim=dim, seed=9, noise=0.0, num_classes=classes,
                       layers=layers, hidden=hidden, eta=0.1, decay=0.0, batch=B,
                       lease_seed=13, partitions=64, init_seed=4)
    joining = rank >= half
    if joining:
        job = rt.Job.joining(cfg, ring0, newcomers, full[rank], local, rank, SWITCH)
    else:
        job = rt.Job(cfg, ring0, [local if r == rank else -1 for r in range(half)])
        job.schedule(SWITCH, True, newcomers, [-1] * len(newcomers))
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    dist.barrier()

    got = {}
    for _ in range(steps):
        rep = job.step()
        if full[rank] in job.ring():
            got[rep.t] = job.sync()
    if sorted(got) != list(range(0 if not joining else SWITCH, steps)):
        failures.append(f"rank {rank}: stepped {sorted(got)}")
    if job.ring() != full:
        failures.append(f"rank {rank}: ring {job.ring()}")
    pj = api.Job(restated(), mspec, 2, 0.0, 0.0, B, 13, 64, ring0)
    pj.schedule(SWITCH, True, newcomers)
    orc = MLPOracle(dim, hidden, classes, layers, 9, 4, 0.1, 0.0)
    for t in range(steps):
        pj.step()
        plan = [(wk, [i for _, i in s]) for wk, s in pj.plan()]
        ref_loss = orc.step(plan, t)
        if t in got and abs(got[t].loss - ref_loss) > 1e-3 * abs(ref_loss):
            failures.append(f"rank {rank}: t={t} loss {got[t].loss} vs {ref_loss}")
        if t in got and got[t].switched != (1 if t == SWITCH else 0):
            failures.append(f"rank {rank}: t={t} switched={got[t].switched}")
    job.gather_master()
    wm = job.params(full[rank])
    ref = orc.flat_master()
    err = np.abs(wm - ref)
    if err.max() > 2 ** -8 * np.abs(ref).max() or err.mean() > 1e-4 * np.abs(ref).max() \
            or np.linalg.norm(err) > 1e-3 * np.linalg.norm(ref):
        failures.append(f"rank {rank}: params max err {err.max()} mean {err.mean()}")
    if job.log_text() != pj.log_text():
        failures.append(f"rank {rank}: assignment log differs")

    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.barrier()
    job.close()
    dist.barrier()
    dist.destroy_process_group()
    flat = [f for fs in allf for f in fs]
    if rank == 0:
        print("MP-SCALE-OUT", "OK" if not flat else "FAIL", flat, flush=True)
    sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
