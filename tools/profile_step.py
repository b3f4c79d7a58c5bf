"""Short, deterministic workload for ncu: the bench's MLP job (BASELINE.json configs[1]),
`--warmup` untimed steps then `--steps` steps, synchronised at the end.

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file profiles/<round>_launches.csv python tools/profile_step.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import WORKLOAD  # noqa: E402
from paper_1909_11985_b200 import runtime as rt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--size", type=int, default=WORKLOAD["size"])
    a = ap.parse_args()
    w = WORKLOAD
    cfg = rt.JobConfig(model=rt.MLP, size=a.size, dim=w["dim"], seed=1, noise=0.0,
                       num_classes=w["classes"], layers=w["layers"], hidden=w["hidden"],
                       eta=0.05, batch=w["batch"], per_worker_batch=w["batch"], lease_seed=7,
                       partitions=64, init_seed=0, keep_log=False)
    job = rt.Job(cfg, ["w00"], [0])
    for _ in range(a.warmup + a.steps):
        job.step()
    rep = job.sync()
    print(f"t={rep.t} loss={rep.loss:.6f} step_ms={rep.step_ms:.3f}")
    job.close()


if __name__ == "__main__":
    main()
