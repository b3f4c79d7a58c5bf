import os, sys, time
sys.path.insert(0, '.')
from paper_1909_11985_b200 import runtime as rt
def trial(batch, width, layers, size=1<<16, ev_t=3, steps=8):
    cfg = rt.JobConfig(model=rt.MLP, size=size, dim=width, seed=1, noise=0.0, num_classes=width,
                       layers=layers, hidden=width, eta=0.05, batch=batch, lease_seed=7, init_seed=0)
    job = rt.Job(cfg, ["w00"], [0])
    job.schedule(ev_t, True, ["w01"], [1])
    try:
        for i in range(steps):
            job.step(); r = job.sync()
        print(f"OK   batch={batch} width={width} layers={layers} last loss {r.loss:.4f}", flush=True)
    except Exception as e:
        print(f"FAIL batch={batch} width={width} layers={layers} at t={i}: {e}", flush=True)
        return False
    finally:
        pass
    job.close()
    return True
cases = [(192, 256, 3), (2048, 256, 3), (192, 4096, 2), (1024, 4096, 2), (2048, 4096, 2), (2048, 4096, 8)]
for c in cases:
    if not trial(*c):
        break
