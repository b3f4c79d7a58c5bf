"""Stall of stop-free scaling with one process per GPU (BASELINE.json configs[2]/[3]).

Run under torch.distributed.run with N (even) processes.  The lower half of the ranks train the
configs[1] MLP (4096 x 8, bf16, constant aggregate batch B); the upper half build their
newcomers with Job.joining while the ring trains (context, HBM dataset, buffers, kernels),
replay the lease protocol host-only and switch in at t=S1 (the ring's processes copy the
consolidated model into them over NVLink); at t=S2 the upper half leaves again (scale-in,
the leavers' processes get Exit).  Every process syncs after each mini-batch so step_ms is
the device time of that mini-batch on its GPU; rank 0 prints, as one JSON line, the max over
the ring's ranks of each mini-batch's time and

  stall_ms = switch mini-batch - median of the following steady mini-batches (same ring),
             each mini-batch counted with the device idle gap before it (the switch's model
             copies are enqueued ahead of its first kernel)

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
      tools/mp_elastic_bench.py [--batch 2048]
"""
import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1909_11985_b200 import runtime as rt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=2048)
    ap.add_argument("--s1", type=int, default=20)
    ap.add_argument("--s2", type=int, default=40)
    ap.add_argument("--steps", type=int, default=60)
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    full = [f"w{r:02d}" for r in range(world)]
    half = world // 2
    ring0, newcomers = full[:half], full[half:]
    cfg = rt.JobConfig(model=rt.MLP, size=1 << 20, dim=4096, seed=1, noise=0.0, num_classes=4096,
                       layers=8, hidden=4096, eta=0.05, batch=args.batch, lease_seed=7,
                       partitions=0, max_workers=world, init_seed=0, keep_log=False)
    if rank >= half:
        job = rt.Job.joining(cfg, ring0, newcomers, full[rank], local, rank, args.s1)
    else:
        job = rt.Job(cfg, ring0, [local if r == rank else -1 for r in range(half)])
        job.schedule(args.s1, True, newcomers, [-1] * len(newcomers))
    job.schedule(args.s2, False, newcomers)
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    dist.barrier()
    ms = {}
    for _ in range(args.steps):
        rep = job.step()
        if full[rank] not in job.ring():
            if rep.t >= args.s2:
                break
            continue
        r2 = job.sync()
        ms[rep.t] = r2.step_ms + r2.stall_ms  # incl. the idle gap of the switch's copies
        if os.environ.get("EDL_STALL_DEBUG") and rep.t in (args.s1 - 1, args.s1, args.s1 + 1,
                                                         args.s2, args.s2 + 1):
            print(f"rank {rank} t={rep.t} step_ms={r2.step_ms:.3f} gap_ms={r2.stall_ms:.3f}",
                  file=sys.stderr, flush=True)
    allms = [None] * world
    dist.all_gather_object(allms, ms)
    dist.barrier()
    job.close()
    if rank == 0:
        per_t = {}
        for m in allms:
            for t, v in m.items():
                per_t[t] = max(per_t.get(t, 0.0), v)

        def stall(s, lo, hi):
            steady = statistics.median(per_t[t] for t in range(lo, hi))
            return per_t[s] - steady, steady

        out_stall, out_steady = stall(args.s1, args.s1 + 3, args.s2)
        in_stall, in_steady = stall(args.s2, args.s2 + 3, args.steps)
        before = statistics.median(per_t[t] for t in range(3, args.s1))
        print(json.dumps({
            "what": "stop-free scaling across processes (one per GPU), MLP 4096x8 bf16",
            "batch": args.batch, "gpus": world,
            f"scale_out_{half}to{world}": {"switch_t": args.s1, "switch_ms": per_t[args.s1],
                                           "steady_ms": out_steady, "stall_ms": out_stall,
                                           "steady_before_ms": before},
            f"scale_in_{world}to{half}": {"switch_t": args.s2, "switch_ms": per_t[args.s2],
                                          "steady_ms": in_steady, "stall_ms": in_stall},
        }), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
