import os, sys, time
sys.path.insert(0, '.')
from paper_1909_11985_b200 import runtime as rt
mode = sys.argv[1]
cfg = rt.JobConfig(model=rt.MLP, size=1<<18, dim=4096, seed=1, noise=0.0, num_classes=4096,
                   layers=8, hidden=4096, eta=0.05, batch=2048, lease_seed=7, init_seed=0, max_workers=2, t_a_ms=500.0)
job = rt.Job(cfg, ["w00"], [0])
for i in range(10):
    job.step(); job.sync()
if mode == "api":
    st = job.scale_out(["w01"], [1])
else:
    st = job.t + 60
    job.schedule(st, True, ["w01"], [1])
print("switch at", st, "now", job.t, flush=True)
try:
    while job.t < st + 10:
        job.step(); r = job.sync()
        if r.switched or job.t % 20 == 0:
            print("t", r.t, "ring", r.ring_size, "step_ms %.2f" % r.step_ms, "stall %.2f" % r.stall_ms, flush=True)
    print("OK", mode, flush=True)
except Exception as e:
    print("FAIL", mode, "at", job.t, e, flush=True)
