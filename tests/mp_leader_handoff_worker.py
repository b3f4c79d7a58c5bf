"""Worker script for tests/test_multigpu_gpu.py::test_multi_process_leader_handoff (run under
torch.distributed.run with 2 processes, one GPU each).

Leader election and handoff (the reference's LeaseStore,
coordination.cpp:26-117) in a one-process-per-GPU job:
  1. rank 0 wins the election (generation 1) and trains alone; it scales rank 1 out;
  2. the leader then scales ITSELF in: at the switch it exits, erases its lease record, and
     rank 1 -- already holding the same t_cur, B and pipeline cursor, since every process
     replays the leader's decisions -- wins the next election (generation 2);
  3. the new leader scales rank 0 back out (rank 0's process re-joins as a newcomer).
Checked against the oracle driving the same three events at the switch steps the run chose:
identical batch assignments, losses and final parameters within 1e-3 relative.
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import api, restated  # noqa: E402
from oracle.mlp import MLPOracle  # noqa: E402
from paper_1909_11985_b200 import runtime as rt  # noqa: E402
from paper_1909_11985_b200.control import ElasticGroup, LeaderLease, wid  # noqa: E402

DIM, HIDDEN, CLASSES, LAYERS, MOM, ETA = 256, 1024, 1024, 3, 0.9, 0.005
T_MAX = 3000


def batch_lines(text, t0):
    out = []
    for ln in text.splitlines():
        f = ln.split()
        if f and f[0] == "batch" and int(f[1]) >= t0:
            out.append(ln)
    return out


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    assert world == 2
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    store = dist.distributed_c10d._get_default_store()
    B = 128
    mspec = {"size": 4000, "dim": DIM, "seed": 9}
    cfg = rt.JobConfig(model=rt.MLP, size=4000, dim=DIM, seed=9, noise=0.0,
                       num_classes=CLASSES, layers=LAYERS, hidden=HIDDEN, eta=ETA, decay=0.0,
                       momentum=MOM, batch=B, lease_seed=13, partitions=64, init_seed=4,
                       max_workers=2, t_a_ms=2.0)
    lease = LeaderLease(store, ttl=10.0)
    g = ElasticGroup(store, rank, [0], t_a_ms=2.0, poll_every=4, lease=lease)
    failures, got, gens, leaders = [], {}, [], []
    out1 = in0 = out0 = None  # switch steps of the three events
    end_t = None
    if rank == 0:
        if not g.elect():
            failures.append("rank 0 lost the first election")
        gens.append(g.generation)
        job = rt.Job(cfg, [wid(0)], [local])
    else:
        job = g.join(cfg, local, timeout_s=240.0)
        out1 = g.last_event[2]
    while job.t < T_MAX:
        rep = job.step()
        if wid(rank) not in job.ring():
            if rep.switched and rank == 0 and in0 is not None and job.t >= in0:
                # 2. the leader left the ring: give up the lease, wait to be scaled back out
                g.leave(job)
                job.close()
                job = g.join(cfg, local, timeout_s=240.0)
                out0 = g.last_event[2]
                end_t = out0 + 10
            continue
        got[rep.t] = job.sync()
        g.notify_batch_end(job)
        ev = g.last_event
        if ev and ev[0] == "out" and ev[1] == [wid(1)]:
            out1 = ev[2]
        if ev and ev[0] == "in":
            in0 = ev[2]
        if ev and ev[0] == "out" and ev[1] == [wid(0)]:
            out0 = ev[2]
            end_t = out0 + 10
        if g.leader == rank and rank not in leaders:
            leaders.append(rank)
            gens.append(getattr(g, "generation", None))
        if end_t is not None and job.t >= end_t:
            break
        if g.leader != rank:
            continue
        # 1. the first leader scales rank 1 out, then itself in
        if rank == 0 and job.t == 3:
            g.scale_out(job, [1])
        if rank == 0 and out1 is not None and in0 is None and job.t >= out1 + 5 \
                and not g.busy(job):
            g.scale_in(job, [0])
        # 3. the new leader scales rank 0 back out
        if rank == 1 and in0 is not None and job.t >= in0 + 6 and out0 is None \
                and not g.busy(job):
            g.scale_out(job, [1 - rank])
        if g.pending is not None:
            time.sleep(0.02)
    if job.t >= T_MAX:
        failures.append(f"rank {rank}: no progress (t={job.t})")
    info = {"rank": rank, "out1": out1, "in0": in0, "out0": out0, "leaders": leaders,
            "gens": gens, "t": job.t}
    infos = [None] * world
    dist.all_gather_object(infos, info)
    print("rank", rank, info, flush=True)
    if rank == 1:
        if leaders != [1] or gens[-1] != 2:
            failures.append(f"rank 1 did not take over as leader (gen {gens})")
        pj = api.Job(restated(), mspec, 2, 0.0, 0.0, B, 13, 64, [wid(0)])
        pj.schedule(out1, True, [wid(1)])
        pj.schedule(in0, False, [wid(0)])
        pj.schedule(out0, True, [wid(0)])
        orc = MLPOracle(DIM, HIDDEN, CLASSES, LAYERS, 9, 4, ETA, 0.0, momentum=MOM)
        for t in range(job.t):
            pj.step()
            ref = orc.step([(wk, [i for _, i in s]) for wk, s in pj.plan()], t)
            if t in got and abs(got[t].loss - ref) > 1e-3 * abs(ref):
                failures.append(f"rank 1 t={t} loss {got[t].loss} vs {ref}")
                break
        if batch_lines(job.log_text(), out1) != batch_lines(pj.log_text(), out1):
            failures.append("rank 1: batch assignments differ from the oracle's")
        job.gather_master()
        w = job.params(wid(1))
        rel = float(np.linalg.norm(w - orc.flat_master()) / np.linalg.norm(orc.flat_master()))
        if rel > 1e-3:
            failures.append(f"params rel L2 {rel}")
        print("MP-HANDOFF events out1", out1, "in0", in0, "out0", out0, "params rel L2", rel,
              flush=True)
    else:
        job.gather_master()
    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.barrier()
    job.close()
    dist.barrier()
    dist.destroy_process_group()
    flat = [f for fs in allf for f in fs]
    if rank == 0:
        print("MP-HANDOFF", "OK" if not flat else "FAIL", flat, flush=True)
    sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
