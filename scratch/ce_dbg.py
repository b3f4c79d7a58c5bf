# debug driver for EDL_AG_DEFER=2: bench-shaped job, synced or pipelined
import os, sys, time
import torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_1909_11985_b200 import runtime as rt
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
hidden, layers, synced = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "sync"
cfg = rt.JobConfig(model=rt.MLP, size=1 << 16, dim=hidden, seed=1, noise=0.0, num_classes=hidden,
                   layers=layers, hidden=hidden, eta=0.05, decay=0.0, batch=512 * world,
                   per_worker_batch=512, lease_seed=7, partitions=0, max_workers=world, init_seed=0,
                   keep_log=False)
ring = [f"w{r:02d}" for r in range(world)]
job = rt.Job(cfg, ring, [local if r == rank else -1 for r in range(world)])
blobs = [None] * world
dist.all_gather_object(blobs, job.export_handles())
for r, b in enumerate(blobs):
    if r != rank: job.import_handles(b)
dist.barrier()
for i in range(8):
    job.step()
    if synced: print(rank, i, job.sync().loss, flush=True)
print(rank, "final", job.sync().loss, flush=True)
