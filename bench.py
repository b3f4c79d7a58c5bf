#!/usr/bin/env python
"""bench.py — samples/sec of EDL's elastic data-parallel SGD step on B200.

Metric (BASELINE.json): samples/sec at 1/2/4/8 B200.  Workload at N=1: BASELINE.json
configs[1] — MLP 4096-wide x 8 layers, bf16, batch 512 per GPU, softmax-CE over 4096 classes,
plain SGD (the reference's sgd_step semantics), HBM-resident synthetic dataset of 2^20 samples
(8 GiB bf16) fed by partition leases.  A "step" is one mini-batch through the public job API:
host lease draws -> H2D lease runs -> gather -> 8 fwd GEMMs -> softmax-CE -> 15 bwd GEMMs ->
fused allreduce + SGD update -> D2H loss.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples/sec at 1/2/4/8 B200; scale-out/in stall ms vs stop-resume"
UNIT = "samples/s"
WORKLOAD = dict(dim=4096, hidden=4096, classes=4096, layers=8, batch=512, size=1 << 20,
                name="mlp4096x8_bf16_b512_sgd")
# BASELINE.json configs[4]: ~1B-param wide MLP (8 x Linear(11264 -> 11264) = 1,015,021,568
# parameters), the allreduce-bound regime; dataset 2^18 samples (5.9 GB bf16) per GPU
WIDE = dict(dim=11264, hidden=11264, classes=11264, layers=8, batch=512, size=1 << 18,
            name="mlp11264x8_bf16_b512_sgd")
WORKLOADS = {"mlp4096x8": WORKLOAD, "wide11264x8": WIDE}


def flops_per_sample(w=WORKLOAD) -> float:
    """6 * params per sample (fwd 2P + dgrad 2P + wgrad 2P; layer-0 dgrad is skipped but
    kept in the algorithmic count like SURVEY.md §8(d))."""
    p = w["dim"] * w["hidden"] + (w["layers"] - 2) * w["hidden"] ** 2 + w["hidden"] * w["classes"]
    return 6.0 * p, p


def _finite(x):
    """JSON has no NaN/inf: an unmeasured figure is emitted as null."""
    if isinstance(x, float) and not math.isfinite(x):
        return None
    if isinstance(x, dict):
        return {k: _finite(v) for k, v in x.items()}
    if isinstance(x, list):
        return [_finite(v) for v in x]
    return x


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.proc or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_step(batch: int, steps: int, w=WORKLOAD):
    """The CPU port of the same MLP step (oracle/mlp.py, numpy/BLAS on every host core):
    the reference has no MLP, so its SGD semantics are restated there."""
    import numpy as np
    from oracle.mlp import MLPOracle
    orc = MLPOracle(w["dim"], w["hidden"], w["classes"], w["layers"], 1, 0, 0.05, 0.0)
    rng = np.random.default_rng(0)
    times = []
    for t in range(steps):
        ids = rng.integers(0, w["size"], size=batch).astype(np.uint64)
        t0 = time.perf_counter()
        orc.step([("w00", ids)], t)
        times.append(time.perf_counter() - t0)
    return times


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import numpy as np  # noqa: F401
    # size each step's sample so the whole --warmup + --steps run stays near 2 minutes
    probe = cpu_reference_step(16, 1)[0]
    per_sample = probe / 16
    budget = float(os.environ.get("EDL_REF_BUDGET_S", "120"))
    batch = int(max(8, min(512, budget / (args.warmup + args.steps) / per_sample)))
    batch = int(os.environ.get("EDL_REF_BATCH", batch))
    times = cpu_reference_step(batch, args.warmup + args.steps)
    timed = times[args.warmup:]
    total = sum(timed)
    value = batch * len(timed) / total
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": {"workload": "mlp4096x8_bf16_b512_sgd",
                                        "parallelism": f"dp{args.gpus}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{batch}-sample mini-batches of the full 4096x8 MLP step "
                                   f"(numpy/BLAS port oracle/mlp.py; the reference has no MLP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank: int, world: int) -> None:
    import torch
    from paper_1909_11985_b200 import runtime as rt

    dist = None
    if world > 1:
        # plumbing only (handle exchange, barriers, max-over-ranks timing); the gradient
        # exchange itself is the fused NVLink peer-memory kernel, not a library collective
        import torch.distributed as dist
        dist.init_process_group("gloo")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    w = WORKLOADS[args.workload]
    cfg = rt.JobConfig(model=rt.MLP, size=w["size"], dim=w["dim"], seed=1, noise=0.0,
                       num_classes=w["classes"], layers=w["layers"], hidden=w["hidden"],
                       eta=0.05, decay=0.0, batch=w["batch"], per_worker_batch=w["batch"],
                       lease_seed=7, partitions=0, max_workers=max(1, world), init_seed=0,
                       keep_log=False)
    ring = [f"w{r:02d}" for r in range(world)]
    job = rt.Job(cfg, ring, [local if r == rank else -1 for r in range(world)])
    if dist is not None:
        blobs = [None] * world
        dist.all_gather_object(blobs, job.export_handles())
        for r, b in enumerate(blobs):
            if r != rank:
                job.import_handles(b)
        dist.barrier()
    stream = torch.cuda.ExternalStream(job.stream_handle())

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        job.step()
    job.sync()
    barrier()

    flops, P = flops_per_sample(w)
    # ---- value: K pipelined steps (inputs HBM-resident), device-timed on the job stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # keep the GPU under the same load around the (short) timed region so the 200 ms
        # clock samples see it: untimed steps for >= 1 s before and 0.5 s after
        t_load = time.time()
        n_pre = 0
        while max_over_ranks(time.time() - t_load) < 1.0:
            for _ in range(20):
                job.step()
            job.sync()
            n_pre += 1
        job.reset_counters()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            job.step()
        job.join()  # the last mini-batch's deferred push collective runs on a side stream
        e1.record(stream)
        torch.cuda.synchronize()
        launches = job.counters()["launches"]  # library kernels of exactly the K timed steps
        barrier()
        # phase breakdown in a separate K-step pass: the phase-boundary events are stream
        # operations between kernels and would cost the timed steps their launch overlap
        job.set_profile(True)
        job.reset_counters()
        for _ in range(args.steps):
            job.step()
        torch.cuda.synchronize()
        job.set_profile(False)
        counters = job.counters()
        barrier()
        t_load = time.time()
        while max_over_ranks(time.time() - t_load) < 0.5:
            for _ in range(20):
                job.step()
            job.sync()
    ms = max_over_ranks(e0.elapsed_time(e1))
    clocks = clk.summary()
    samples = w["batch"] * args.steps * world
    value = samples / (ms / 1e3)

    ph = counters["phase_ms"]
    n = max(1, counters["steps"])
    wgrad_ms = ph.get("wgrad", 0.0) / n  # the 8 weight-gradient GEMMs (sub-phase of backward)
    ph_main = {k: v for k, v in ph.items() if k != "wgrad"}
    gemm_ms = (ph["forward"] + ph["backward"]) / n
    upd_ms = ph["update"] / n
    gemm_tflops = flops * w["batch"] / (gemm_ms / 1e3) / 1e12
    peaks = measured_peaks()
    peak_t = peaks.get("bf16_tflops_sustained", 1354.1)
    peak_h = peaks.get("hbm_gbs", 6555.5)
    if world == 1:
        # update fused into the weight-gradient GEMM epilogues: 4 B master read + 4 B
        # master write + 2 B bf16 weight write per parameter, inside the backward phase
        upd = {"bound": "hbm", "where": "fused into wgrad GEMM epilogue (backward phase)",
               "bytes_per_step": 10 * P}
    else:
        # allreduce bus bytes per GPU per direction (bf16 reduce-scatter + all-gather,
        # 2(N-1)/N x 2P); the exchange's halves are timed where they run
        mode = job.exchange_mode()
        half = (world - 1) / world * 2 * P
        if mode == 3:
            # reduce-scatter stored from the wgrad GEMM epilogues (inside the backward): only
            # the all-gather half (push collective: shard sum + SGD + weight stores) is exposed
            upd = {"bound": "nvlink", "achieved": half / (upd_ms / 1e3) / 1e9, "peak": 770.0,
                   "unit": "GB/s", "frac": half / (upd_ms / 1e3) / 1e9 / 770.0,
                   "bytes_per_step": half, "per_step_ms": upd_ms,
                   "allreduce_bus_bytes_per_step": 2 * half,
                   "exposed_allreduce_bus_gbs": 2 * half / (upd_ms / 1e3) / 1e9,
                   "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction "
                                  "(900 GB/s NVLink 5 nominal)",
                   "kernel": "push all-gather + sharded SGD (reduce-scatter routed from the "
                             "wgrad GEMM epilogues, overlapped with the backward)"}
        else:
            nv = 2 * half
            upd = {"bound": "nvlink", "achieved": nv / (upd_ms / 1e3) / 1e9, "peak": 770.0,
                   "unit": "GB/s", "frac": nv / (upd_ms / 1e3) / 1e9 / 770.0,
                   "bytes_per_step": nv, "per_step_ms": upd_ms,
                   "allreduce_bus_bytes_per_step": nv,
                   "exposed_allreduce_bus_gbs": nv / (upd_ms / 1e3) / 1e9,
                   "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction "
                                  "(900 GB/s NVLink 5 nominal)",
                   "kernel": "fused reduce-scatter + sharded SGD + all-gather over NVLink P2P"}
        upd["exchange_mode"] = mode

    # ---- roofline of the dominant kernel (profiles/r01_kernel_shares.md): at N=1 the fused
    # weight-gradient GEMM + SGD update (51% of the step), HBM-bound: per launch (one layer,
    # SURVEY 8(d)'s 10 B/param update) 10 B x 16.8M params + its two bf16 operands
    # dY [b][4096] and X [b][4096]; duration = the wgrad sub-phase / 8 launches, CUDA events
    # on the job stream.  With several GPUs the weight-gradient GEMMs write bf16 gradients
    # (tensor-bound) and the update moves to the NVLink collective (update_roofline).
    n_wgrad = w["layers"]
    per_launch_ms = wgrad_ms / n_wgrad if wgrad_ms > 0 else float("nan")
    if world == 1:
        alg = 10 * (P // n_wgrad) + 2 * 2 * w["batch"] * w["hidden"]
        gbs = alg / (per_launch_ms / 1e3) / 1e9
        dominant = {"bound": "hbm", "kernel": "gemm_bf16_2sm_kernel<128,MN,MN,sgd> "
                    "(weight gradient + fused SGD update, one launch per layer)",
                    "achieved": gbs, "peak": peak_h, "unit": "GB/s", "frac": gbs / peak_h,
                    "traffic": _ncu_traffic("wgrad+sgd") if w is WORKLOAD else None,
                    "traffic_source": NCU_FULL,
                    "algorithmic_bytes_per_launch": alg, "launch_ms": per_launch_ms,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)"}
    else:
        tf = 2 * w["batch"] * (P // n_wgrad) / (per_launch_ms / 1e3) / 1e12
        rs = upd.get("exchange_mode") == 3
        dominant = {"bound": "tensor", "kernel": "gemm_bf16_2sm_kernel<128,MN,MN> "
                    + ("(weight gradient, reduce-scatter stored to the shard owners over NVLink "
                       "from the epilogue, one launch per layer)" if rs else
                       "(weight gradient, bf16 out, one launch per layer)"),
                    "achieved": tf, "peak": peak_t, "unit": "TFLOP/s", "frac": tf / peak_t,
                    "traffic": _ncu_traffic("wgrad]") if w is WORKLOAD else None,
                    "traffic_source": NCU_FULL,
                    "algorithmic_flop_per_launch": 2 * w["batch"] * (P // n_wgrad),
                    "launch_ms": per_launch_ms,
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}
        if rs:
            # the epilogue stores the (N-1)/N of each layer's bf16 gradient owned by the other
            # replicas over NVLink: that store stream, not the tensor pipe, bounds the launch
            remote = (world - 1) / world * 2 * (P // n_wgrad)
            dominant["nvlink_store"] = {
                "bytes_per_launch": remote, "achieved": remote / (per_launch_ms / 1e3) / 1e9,
                "peak": 770.0, "unit": "GB/s",
                "frac": remote / (per_launch_ms / 1e3) / 1e9 / 770.0,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}

    # ---- e2e: every step through the public API with a D2H read of its loss
    job.reset_counters()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e2.record(stream)
    losses = []
    for _ in range(args.steps):
        job.step()
        losses.append(job.sync().loss)
    job.join()
    e3.record(stream)
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks(e2.elapsed_time(e3))
    e2e_value = samples / (ms_e2e / 1e3)
    runs_per_step = 2  # a 512-sample batch spans <= 2 shards of >= 4096 samples

    # ---- NCCL baseline for the exchange (N > 1): a library allreduce of the same bf16
    # gradient bytes on the same GPUs, timed like the step (device events, max over ranks);
    # the product path never calls it -- it is the yardstick for the fused NVLink exchange
    if world > 1 and not args.no_nccl:
        try:
            import torch.distributed as dist_
            g = dist_.new_group(backend="nccl")
            buf = torch.zeros(P, dtype=torch.bfloat16, device=f"cuda:{local}")
            for _ in range(3):
                dist_.all_reduce(buf, group=g)
            barrier()
            n_it = 10
            e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e4.record()
            for _ in range(n_it):
                dist_.all_reduce(buf, group=g)
            e5.record()
            torch.cuda.synchronize()
            nms = max_over_ranks(e4.elapsed_time(e5)) / n_it
            upd["nccl_allreduce_same_bytes"] = {
                "ms": nms, "bytes": 2 * P,
                "bus_gbs": 2.0 * (world - 1) / world * 2 * P / (nms / 1e3) / 1e9,
                "note": "torch.distributed NCCL all_reduce(sum) of the bf16 gradient (2P bytes) "
                        "on the same GPUs; compare with the exposed exchange per_step_ms"}
            del buf
            dist_.destroy_process_group(g)
        except Exception as e:  # noqa: BLE001 -- a missing NCCL must not fail the bench
            upd["nccl_allreduce_same_bytes"] = {"unavailable": str(e)[:200]}

    # ---- CPU baseline (oracle port), bounded sample on this host, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and w is WORKLOAD:
        batch = int(os.environ.get("EDL_CPU_BATCH", "64"))
        t = cpu_reference_step(batch, 2)
        cpu = {"value": batch / min(t), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"best of 2 {batch}-sample steps of the full 4096x8 MLP "
                         f"(numpy/BLAS, oracle/mlp.py); the reference has no MLP"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (HBM-resident 2^20 x 4096 bf16 splitmix64 dataset, random-init MLP)",
        "config": {"workload": w["name"], "layers": w["layers"],
                   "width": w["hidden"], "classes": w["classes"],
                   "global_batch": samples // args.steps, "per_gpu_batch": w["batch"],
                   "dataset_samples": w["size"], "parallelism": f"dp{world}",
                   "optimizer": "sgd(eta=0.05), fp32 master",
                   "l2": "inputs > L2 (weights 268 MB + fp32 master 537 MB streamed per step)"},
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": 16 * runs_per_step, "d2h_bytes_per_step": 8,
                "note": "job.step()+job.sync() per step: host lease draws, the lease runs "
                        "H2D as gather-kernel launch parameters, D2H loss"},
        "gpu_launches": launches,
        "roofline": dominant,
        "gemm_roofline": {"bound": "tensor", "kernel": "tcgen05 GEMMs (8 fwd + 7 dgrad + 8 wgrad)",
                          "achieved": gemm_tflops, "peak": peak_t, "unit": "TFLOP/s",
                          "frac": gemm_tflops / peak_t,
                          "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                          "per_step_ms": gemm_ms,
                          "algorithmic_gflop_per_step": flops * w["batch"] / 1e9},
        "update_roofline": upd,
        "phase_ms_per_step": {k: v / n for k, v in ph_main.items()},
        "wgrad_ms_per_step": wgrad_ms,
        "loss_first_last": [losses[0], losses[-1]] if losses else None,
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(_finite(line)), flush=True)
    if dist is not None:
        dist.barrier()
    job.close()
    if dist is not None:
        dist.destroy_process_group()


NCU_FULL = "profiles/r01_ncu_full.md"


def _ncu_traffic(family: str):
    """Mean DRAM read + write bytes per launch of a kernel family in the committed
    ncu --set full capture (profiles/r01_ncu_full.md), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), NCU_FULL)
    vals = []
    try:
        for line in open(path):
            cells = [c.strip() for c in line.split("|")]
            if len(cells) > 5 and family in cells[2]:
                vals.append((float(cells[4]) + float(cells[5])) * 1e6)
    except (OSError, ValueError):
        return None
    return sum(vals) / len(vals) if vals else None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-nccl", action="store_true",
                    help="skip the NCCL allreduce yardstick at N > 1")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="mlp4096x8",
                    help="mlp4096x8 = BASELINE configs[1] (the headline); wide11264x8 = "
                         "configs[4], the ~1B-param allreduce-bound MLP")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world)


if __name__ == "__main__":
    main()
