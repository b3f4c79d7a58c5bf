"""Noise floor of the MLP parity tests: how far two *valid* fp32
implementations of the same bf16 MLP SGD step drift apart when they differ only in GEMM
accumulation order.  The oracle (oracle/mlp.py, fp32 BLAS) is run twice on the lease plans of
tests/test_headline_parity_gpu.py: once as is, once with every GEMM accumulated in f64 and
rounded to fp32.  bf16 rounding flips of the activations then propagate through the 8 layers,
which sets the smallest tolerance any GPU implementation can be held to.

  python tools/parity_floor.py [--steps 6] [--width 4096]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import api, restated  # noqa: E402
from oracle import mlp as om  # noqa: E402

_MM = torch.Tensor.__matmul__


def plans(events, steps, size, width, B=512):
    spec = {"size": size, "dim": width, "seed": 1, "noise": 0.0, "sign_labels": False}
    job = api.Job(restated(), spec, 2, 0.0, 0.0, B, 7, 64, ["w00"])
    for t, out, ids in events:
        job.schedule(t, out, ids)
    out = []
    for _ in range(steps):
        job.step()
        out.append([(w, [i for _, i in s]) for w, s in job.plan()])
    return out


def run(ps, f64_accumulate, mom, eta, width):
    o = om.MLPOracle(width, width, width, 8, 1, 0, eta, 0.0, momentum=mom)
    w0 = o.flat_master().copy()
    if f64_accumulate:
        torch.Tensor.__matmul__ = lambda a, b: _MM(a.double(), b.double()).float()
    try:
        losses = [o.step(p, t) for t, p in enumerate(ps)]
    finally:
        torch.Tensor.__matmul__ = _MM
    return w0, o.flat_master(), losses


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--width", type=int, default=4096)
    args = ap.parse_args()
    events = [(2, True, ["w01"]), (4, False, ["w00"])]
    ps = plans(events, args.steps, 1 << 20, args.width)
    for mom, eta in ((0.0, 0.05), (0.9, 0.05), (0.9, 0.005)):
        w0, a, la = run(ps, False, mom, eta, args.width)
        _, b, lb = run(ps, True, mom, eta, args.width)
        print(json.dumps({
            "momentum": mom, "eta": eta, "steps": args.steps, "width": args.width,
            "loss_rel_max": max(abs(x - y) / abs(y) for x, y in zip(la, lb)),
            "params_rel_l2": float(np.linalg.norm(a - b) / np.linalg.norm(b)),
            "update_rel_l2": float(np.linalg.norm(a - b) / np.linalg.norm(b - w0)),
            "update_over_params": float(np.linalg.norm(b - w0) / np.linalg.norm(b))}))


if __name__ == "__main__":
    main()
