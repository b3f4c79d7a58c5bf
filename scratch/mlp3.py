import numpy as np, sys
sys.path.insert(0, '.')
from oracle import api, restated
from oracle.mlp import MLPOracle
from paper_1909_11985_b200 import runtime as rt
dim, hidden, classes, layers, B = 64, 128, 64, 3, 96
spec = {"size": 3000, "dim": dim, "seed": 5}
for fail in (False, True):
  for ring in (["w00"], ["w00","w01"], ["w00","w01","w02"]):
    cfg = rt.JobConfig(model=rt.MLP, size=3000, dim=dim, seed=5, noise=0.0, num_classes=classes,
                       layers=layers, hidden=hidden, eta=0.1, decay=0.01, batch=B,
                       lease_seed=11, partitions=64, init_seed=3, appx_recovery=True)
    job = rt.Job(cfg, ring, [0]*len(ring))
    pj = api.Job(restated(), spec, 2, 0.0, 0.0, B, 11, 64, ring)
    orc = MLPOracle(dim, hidden, classes, layers, 5, 3, 0.1, 0.01)
    errs = []
    for t in range(16):
        if fail and t == 10 and len(ring) > 1:
            job.fail([ring[-1]], approximate=True); pj.fail_approximate([ring[-1]]); orc.master = [m.copy() for m in saved]
            t = 9
        job.step(); pj.step()
        saved = [m.copy() for m in orc.master]
        orc.step([(wk, [i for _, i in s]) for wk, s in pj.plan()], job.t - 1)
        job.sync()
        w = job.params(job.ring()[0]); ref = orc.flat_master()
        errs.append(np.abs(w - ref).max() / np.abs(ref).max())
    print("fail" if fail else "plain", len(ring), ["%.1e" % e for e in errs[::3]], "final %.2e" % errs[-1])
