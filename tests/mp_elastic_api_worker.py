"""Worker script for tests/test_multigpu_gpu.py::test_multi_process_scheduler_facing_scaling
(run under torch.distributed.run, one process per GPU).

The scheduler-facing elastic API across processes, driven through
the control plane of paper_1909_11985_b200/control.py over the rendezvous TCPStore:

  * rank 0 trains alone (MLP, momentum 0.9); at t=3 the scheduler calls scale_out(others):
    the idle processes build their newcomers while rank 0 keeps training, report Ready, and
    the leader fixes switch_t = t_ready + max(k, margin); a second scale_out / scale_in while
    that is pending must answer Retry;
  * after the switch the newcomers run with the ring (momentum buffers copied in with the
    model); rank 1 is then slowed by an injected delay, every process publishes its worker's
    mini-batch times, the leader's straggler rule (1.2x the median for 10 mini-batches)
    names rank 1 and the leader scales the newcomers in again.

Checked against the CPU oracle driving the same events at the switch steps the run chose:
identical assignment log, loss trajectory and parameters within 1e-3 relative.
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
from paper_1909_11985_b200 import _lib  # noqa: E402
from paper_1909_11985_b200 import runtime as rt  # noqa: E402
from paper_1909_11985_b200.control import ElasticGroup, wid  # noqa: E402

T_MAX = 4000
DIM, HIDDEN, CLASSES, LAYERS = 256, 1024, 1024, 3
MOM, ETA = 0.9, 0.005


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    store = dist.distributed_c10d._get_default_store()
    B = 64 * world
    mspec = {"size": 4000, "dim": DIM, "seed": 9}
    cfg = rt.JobConfig(model=rt.MLP, size=4000, dim=DIM, seed=9, noise=0.0,
                       num_classes=CLASSES, layers=LAYERS, hidden=HIDDEN, eta=ETA, decay=0.0,
                       momentum=MOM, batch=B, lease_seed=13, partitions=64, init_seed=4,
                       max_workers=world, t_a_ms=2.0)
    g = ElasticGroup(store, rank, [0], t_a_ms=2.0, poll_every=4)
    others = list(range(1, world))
    failures, events, got = [], [], {}
    retry_seen = {"out": False, "in": False}
    straggler_at = None

    if rank == 0:
        job = rt.Job(cfg, [wid(0)], [local])
    else:
        job = g.join(cfg, local, timeout_s=240.0)
    out_switch = in_switch = None
    while job.t < T_MAX:
        rep = job.step()
        if wid(rank) not in job.ring():
            if rank != 0 and rep.switched and out_switch is not None:
                break  # scaled in: notify_batch_end answered Exit
            continue  # newcomer before its switch: host-only replay
        got[rep.t] = job.sync()
        ev = g.notify_batch_end(job)
        if ev is not None:
            events.append(ev)
        if g.last_event and g.last_event[0] == "out":
            out_switch = g.last_event[2]
        if g.last_event and g.last_event[0] == "in":
            in_switch = g.last_event[2]
        if rank == 0 and in_switch is not None and job.t >= in_switch + 8:
            break
        # scheduler (rank 0): scale_out at t=3, Retry while it is pending
        if rank == 0 and job.t == 3:
            if g.scale_out(job, others) != -1:
                failures.append("scale_out did not return pending (-1)")
        elif rank == 0 and job.t == 4:
            for kind, fn in (("out", g.scale_out), ("in", g.scale_in)):
                try:
                    fn(job, others)
                except _lib.EdlError as e:
                    retry_seen[kind] = e.code == _lib.EDL_RETRY
        if rank == 0 and g.pending is not None:
            time.sleep(0.02)  # the ring keeps training (slowly) while the newcomers build
        # straggler: rank 1 slowed after the switch; every ring process publishes its times
        if out_switch is not None and job.t > out_switch + 2 and in_switch is None:
            if rank == 1 and job.t == out_switch + 3:
                job.set_worker_delay(wid(1), 400.0)
            g.publish_times(job, 10)
            if rank == 0 and straggler_at is None and not g.busy(job):
                s = g.straggler(10, 1.2)
                if s is not None:
                    straggler_at = job.t
                    if s != 1:
                        failures.append(f"straggler rule named rank {s}")
                    sw = g.scale_in(job, others)
                    events.append(("in", [wid(r) for r in others], sw))
    if job.t >= T_MAX:
        failures.append(f"rank {rank}: no progress to the end (t={job.t})")
    print(f"rank {rank} done at t={job.t} events={events}", flush=True)
    if rank == 0:
        if not all(retry_seen.values()):
            failures.append(f"no Retry while pending: {retry_seen}")
        if straggler_at is None:
            failures.append("straggler never detected")
        outs = [e for e in events if e[0] == "out"]
        ins = [e for e in events if e[0] == "in"]
        if len(outs) != 1 or len(ins) != 1:
            failures.append(f"events {events}")
        else:
            # the oracle drives the same events at the switch steps the run chose
            pj = api.Job(restated(), mspec, 2, 0.0, 0.0, B, 13, 64, [wid(0)])
            pj.schedule(outs[0][2], True, outs[0][1])
            pj.schedule(ins[0][2], False, ins[0][1])
            orc = MLPOracle(DIM, HIDDEN, CLASSES, LAYERS, 9, 4, ETA, 0.0, momentum=MOM)
            for t in range(job.t):
                pj.step()
                ref = orc.step([(wk, [i for _, i in s]) for wk, s in pj.plan()], t)
                if abs(got[t].loss - ref) > 1e-3 * abs(ref):
                    failures.append(f"t={t} loss {got[t].loss} vs {ref}")
                    break
            if job.log_text() != pj.log_text():
                failures.append("assignment log differs from the oracle's")
            w = job.params(wid(0))
            refw = orc.flat_master()
            rel = float(np.linalg.norm(w - refw) / np.linalg.norm(refw))
            if rel > 1e-3:
                failures.append(f"params rel L2 {rel}")
            print("MP-ELASTIC-API events", events, "straggler detected at t", straggler_at,
                  "params rel L2", rel, flush=True)
            if job.ring() != [wid(0)]:
                failures.append(f"ring {job.ring()}")
    allf = [None] * world
    dist.all_gather_object(allf, failures)
    dist.barrier()
    job.close()
    dist.barrier()
    dist.destroy_process_group()
    flat = [f for fs in allf for f in fs]
    if rank == 0:
        print("MP-ELASTIC-API", "OK" if not flat else "FAIL", flat, flush=True)
    sys.exit(1 if flat else 0)


if __name__ == "__main__":
    main()
