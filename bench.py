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


def flops_per_sample(w=WORKLOAD):
    """GEMM FLOPs per sample of the GEMMs the step runs, and the parameter count P.
    fwd 2P + wgrad 2P + dgrad 2(P - P_0): the layer-0 dgrad (the gradient w.r.t. the input
    features) is never computed, so it is not counted (SURVEY.md §8(d)'s 6P counts it)."""
    p0 = w["dim"] * w["hidden"]
    p = p0 + (w["layers"] - 2) * w["hidden"] ** 2 + w["hidden"] * w["classes"]
    return 6.0 * p - 2.0 * p0, p


def fwd_dgrad_flops_per_sample(w=WORKLOAD) -> float:
    """The tensor-bound GEMMs: 8 forward + 7 dgrad (the wgrad GEMMs carry the fused update
    at N=1 and are timed as the dominant, HBM-bound kernel)."""
    fl, p = flops_per_sample(w)
    return fl - 2.0 * p


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


def cpu_mlp_port_steps(batch: int, steps: int, w=WORKLOAD):
    """The CPU port of the same MLP step (oracle/mlp.py: torch CPU fp32 BLAS on every host
    core, the GPU's bf16 rounding points): the reference has no MLP, so its
    SGD semantics are restated there.  Returns per-step seconds."""
    import numpy as np
    import torch
    from oracle.mlp import MLPOracle
    torch.set_num_threads(os.cpu_count() or 1)
    orc = MLPOracle(w["dim"], w["hidden"], w["classes"], w["layers"], 1, 0, 0.05, 0.0)
    rng = np.random.default_rng(0)
    times = []
    for t in range(steps):
        ids = rng.integers(0, w["size"], size=batch).astype(np.uint64)
        t0 = time.perf_counter()
        orc.step([("w00", ids)], t)
        times.append(time.perf_counter() - t0)
    return times


LINEAR = dict(size=8192, dim=4096, batch=512, eta=0.05, name="linear_ls_dim4096_b512")


def reference_linear(budget_s: float = 6.0):
    """The reference's own CPU path, compiled from /root/reference (oracle/_ref/libedlref.so),
    on the linear least-squares job at dim 4096 / batch 512: per step
    SyntheticDataset::get x 512 (dataset.cpp:36-54) + local_gradient (trainer.cpp:30-39) +
    sgd_step (trainer.cpp:56-61) behind the reference ShardManager (datapipeline.cpp), one
    thread (the reference runs one thread per worker; one worker here)."""
    from oracle import api, reference
    R = reference()
    if R is None:
        return {"unavailable": "oracle/_ref/libedlref.so not built (needs /root/reference)"}
    spec = {"size": LINEAR["size"], "dim": LINEAR["dim"], "seed": 1, "noise": 0.01,
            "sign_labels": False}
    job = api.Job(R, spec, 0, LINEAR["eta"], 0.0, LINEAR["batch"], 7, 64, ["w00"])
    job.step()  # warm-up
    n, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s or n < 3:
        job.step()
        n += 1
    dt = time.perf_counter() - t0
    return {"value": LINEAR["batch"] * n / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "ms_per_step": 1e3 * dt / n, "workload": LINEAR["name"],
            "sample": f"{n} mini-batches of the reference's linear job (SyntheticDataset dim "
                      f"4096, batch 512, ShardManager leases, local_gradient + sgd_step), "
                      f"compiled from /root/reference by oracle/Makefile"}


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    times = cpu_mlp_port_steps(w["batch"], args.warmup + args.steps, w)
    timed = times[args.warmup:]
    total = sum(timed)
    value = w["batch"] * len(timed) / total
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic", "config": {"workload": w["name"], "global_batch": w["batch"],
                                        "per_gpu_batch": w["batch"], "parallelism": "cpu",
                                        "same_config": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{len(timed)} full {w['batch']}-sample mini-batches of the "
                                   f"{w['name']} step (torch CPU fp32 BLAS port oracle/mlp.py "
                                   f"on {cores} threads; the reference has no MLP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_linear": reference_linear(),
    }
    print(json.dumps(_finite(line)), flush=True)


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
    # the phase breakdown comes from the profiled pass (events at phase boundaries break the
    # PDL launch overlap, so its phases sum to more than the unprofiled step); every per-step
    # figure below is that phase's SHARE of the profiled step times the unprofiled ms/step
    prof_ms = sum(v for k, v in ph.items() if k != "wgrad") / n
    share = (ms / args.steps) / prof_ms if prof_ms > 0 else float("nan")
    wgrad_ms = ph.get("wgrad", 0.0) / n  # the 8 weight-gradient GEMMs (sub-phase of backward)
    ph_main = {k: v for k, v in ph.items() if k != "wgrad"}
    fd_ms = (ph["forward"] + ph["backward"]) / n - wgrad_ms  # 8 fwd + 7 dgrad GEMMs
    upd_ms = ph["update"] / n
    fd_flops = fwd_dgrad_flops_per_sample(w) * w["batch"]
    gemm_tflops = fd_flops / (fd_ms * share / 1e3) / 1e12
    peaks = measured_peaks()
    peak_t = peaks.get("bf16_tflops_sustained", 1354.1)
    peak_h = peaks.get("hbm_gbs", 6555.5)
    # split master (the library's default, EDL_SPLIT_MASTER=0 turns it off): the fused update
    # reads and writes the bf16 weights W and the low 16 bits of the fp32 master, 8 B/param;
    # the fp32 master itself: 4 B read + 4 B write + 2 B bf16 weight write = 10 B/param
    upd_bpp = 8 if os.environ.get("EDL_SPLIT_MASTER", "1") != "0" else 10
    if world == 1:
        upd = {"bound": "hbm", "where": "fused into wgrad GEMM epilogue (backward phase)",
               "bytes_per_param": upd_bpp, "bytes_per_step": upd_bpp * P}
    else:
        # allreduce bus bytes per GPU per direction (bf16 reduce-scatter + all-gather,
        # 2(N-1)/N x 2P); the exchange's halves are timed where they run
        mode = job.exchange_mode()
        half = (world - 1) / world * 2 * P
        if mode in (3, 5, 6):
            # reduce-scatter stored from the wgrad GEMM epilogues (mode 3) or copied by the copy
            # engines layer by layer (mode 5), inside the backward: only the all-gather half
            # (push collective: shard sum + SGD + weight stores) is exposed
            rs_ms = wgrad_ms if mode == 3 else ph["backward"] / n  # 5 / 6: under the backward
            upd = {"bound": "nvlink", "achieved": half / (upd_ms / 1e3) / 1e9, "peak": 770.0,
                   "unit": "GB/s", "frac": half / (upd_ms / 1e3) / 1e9 / 770.0,
                   "bytes_per_step": half, "per_step_ms": upd_ms * share,
                   "allreduce_bus_bytes_per_step": 2 * half,
                   # bus bandwidth: RS + AG bytes over the time the transfers occupy (the
                   # reduce-scatter rides in the wgrad GEMMs / the backward, the all-gather is
                   # the push)
                   "busbw_gbs": 2 * half / ((rs_ms + upd_ms) / 1e3) / 1e9,
                   "busbw_peak_gbs": 900.0,
                   "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction "
                                  "(900 GB/s NVLink 5 nominal)",
                   "kernel": "push all-gather + sharded SGD (reduce-scatter "
                             + {3: "routed from the wgrad GEMM epilogues",
                                5: "on the copy engines, layer by layer",
                                6: "split between the wgrad GEMM epilogues and the copy engines"}[mode] +
                             ", overlapped with the backward)"}
        else:
            nv = 2 * half
            upd = {"bound": "nvlink", "achieved": nv / (upd_ms / 1e3) / 1e9, "peak": 770.0,
                   "unit": "GB/s", "frac": nv / (upd_ms / 1e3) / 1e9 / 770.0,
                   "bytes_per_step": nv, "per_step_ms": upd_ms * share,
                   "allreduce_bus_bytes_per_step": nv,
                   "busbw_gbs": nv / (upd_ms / 1e3) / 1e9, "busbw_peak_gbs": 900.0,
                   "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction "
                                  "(900 GB/s NVLink 5 nominal)",
                   "kernel": "fused reduce-scatter + sharded SGD + all-gather over NVLink P2P"}
        upd["exchange_mode"] = mode

    # ---- roofline of the dominant kernel (profiles/r02_kernel_shares.md): at N=1 the fused
    # weight-gradient GEMM + SGD update (~45% of the step), HBM-bound: per launch (one layer)
    # 8 B/param over the split master (10 B with the fp32 one) x 16.8M params + its two bf16
    # operands
    # dY [b][4096] and X [b][4096]; duration = the wgrad sub-phase / 8 launches, CUDA events
    # on the job stream.  With several GPUs the weight-gradient GEMMs write bf16 gradients
    # (tensor-bound) and the update moves to the NVLink collective (update_roofline).
    n_wgrad = w["layers"]
    per_launch_ms = wgrad_ms / n_wgrad if wgrad_ms > 0 else float("nan")
    if world == 1:
        alg = upd_bpp * (P // n_wgrad) + 2 * 2 * w["batch"] * w["hidden"]
        gbs = alg / (per_launch_ms / 1e3) / 1e9
        dominant = {"bound": "hbm", "kernel": "gemm_bf16_2sm_kernel<128,MN,MN,sgd> "
                    "(weight gradient + fused SGD update, one launch per layer)",
                    "achieved": gbs, "peak": peak_h, "unit": "GB/s", "frac": gbs / peak_h,
                    "traffic": _ncu_traffic("wgrad+sgd") if w is WORKLOAD else None,
                    "traffic_source": NCU_STEP,
                    "algorithmic_bytes_per_launch": alg, "bytes_per_param": upd_bpp,
                    "launch_ms": per_launch_ms,
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
    cpu = ref_lin = None
    if rank == 0 and world == 1 and not args.no_cpu and w is WORKLOAD:
        steps_cpu = int(os.environ.get("EDL_CPU_STEPS", "3"))
        t = cpu_mlp_port_steps(w["batch"], steps_cpu + 1, w)[1:]
        cpu = {"value": w["batch"] * len(t) / sum(t), "unit": UNIT, "cores": os.cpu_count(),
               "kind": "port",
               "sample": f"{len(t)} full {w['batch']}-sample mini-batches of the 4096x8 MLP "
                         f"step after one warm-up (torch CPU fp32 BLAS port oracle/mlp.py, "
                         f"{os.cpu_count()} threads); the reference has no MLP"}
        ref_lin = reference_linear()

    # ---- the reference's own path on the GPU: the linear least-squares job at dim 4096 /
    # batch 512 through the same job API, f64, bit-exact with the reference
    lin = None
    if rank == 0 and world == 1 and not args.no_cpu:
        lin = gpu_linear_job(args.steps)
        if ref_lin and ref_lin.get("value"):
            lin["reference_cpu"] = ref_lin
            lin["speedup_vs_reference"] = lin["value"] / ref_lin["value"]

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
        "gemm_roofline": {"bound": "tensor", "kernel": "tcgen05 GEMMs (8 fwd + 7 dgrad)",
                          "achieved": gemm_tflops, "peak": peak_t, "unit": "TFLOP/s",
                          "frac": gemm_tflops / peak_t,
                          "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                          "per_step_ms": fd_ms * share,
                          "algorithmic_gflop_per_step": fd_flops / 1e9,
                          "note": "per_step_ms = the fwd+dgrad share of the profiled pass x the "
                                  "unprofiled ms_per_step"},
        "step_tflops": {"achieved": flops * w["batch"] / (ms / args.steps / 1e3) / 1e12,
                        "gflop_per_step": flops * w["batch"] / 1e9, "gemms": 23,
                        "frac": flops * w["batch"] / (ms / args.steps / 1e3) / 1e12 / peak_t,
                        "note": "all GEMM FLOPs of the step over the whole step time"},
        "update_roofline": upd,
        "phase_ms_per_step_profiled": {k: v / n for k, v in ph_main.items()},
        "wgrad_ms_per_step_profiled": wgrad_ms,
        "profiled_over_unprofiled": 1.0 / share,
        "loss_first_last": [losses[0], losses[-1]] if losses else None,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "linear_job": lin,
    }
    if dist is not None:
        dist.barrier()
    job.close()
    # ---- stop-free scaling stall vs stop-resume (the metric's second half, configs[2]/[3])
    if not args.no_elastic and w is WORKLOAD:
        line["elastic"] = (elastic_leg_single(args) if world == 1 else
                           elastic_leg_mp(args, rank, world, local, dist))
    if rank == 0:
        print(json.dumps(_finite(line)), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def gpu_linear_job(steps: int) -> dict:
    """LeastSquares job at dim 4096 / batch 512 on cuda:0 through the public job API (the f64
    kernels that reproduce trainer.cpp bit for bit), timed with CUDA events."""
    import torch
    from paper_1909_11985_b200 import runtime as rt
    cfg = rt.JobConfig(model=rt.LEAST_SQUARES, size=LINEAR["size"], dim=LINEAR["dim"], seed=1,
                       noise=0.01, eta=LINEAR["eta"], batch=LINEAR["batch"], lease_seed=7,
                       partitions=64, keep_log=False)
    job = rt.Job(cfg, ["w00"], [0])
    for _ in range(5):
        job.step()
    job.sync()
    stream = torch.cuda.ExternalStream(job.stream_handle())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        job.step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    job.close()
    return {"workload": LINEAR["name"], "value": LINEAR["batch"] * steps / (ms / 1e3),
            "unit": UNIT, "ms_per_step": ms / steps, "dtype": "f64",
            "note": "GPU f64 path bit-exact with the reference trainer (tests/test_job_gpu.py); "
                    "latency-bound sequential sums, not a throughput kernel"}


def _elastic_cfg(batch: int, world: int):
    from paper_1909_11985_b200 import runtime as rt
    w = WORKLOAD
    return rt.JobConfig(model=rt.MLP, size=w["size"], dim=w["dim"], seed=1, noise=0.0,
                        num_classes=w["classes"], layers=w["layers"], hidden=w["hidden"],
                        eta=0.05, batch=batch, lease_seed=7, partitions=0,
                        max_workers=max(2, world), init_seed=0, t_a_ms=500.0, keep_log=True)


def _switch_stall(reps, settle: int = 10) -> dict:
    """reps: per-mini-batch reports (synced each step) around one switch.  A mini-batch's
    device cost is its own time plus the device idle gap before it (the model copies and
    consolidation of a switch are enqueued before the switch mini-batch's first kernel);
    stall = that cost at the switch minus its median over the steady mini-batches after."""
    k = next(i for i, r in enumerate(reps) if r.switched)
    cost = [r.step_ms + r.stall_ms for r in reps]
    before = statistics.median(cost[max(0, k - settle):k])
    after = statistics.median(cost[k + 2:k + 2 + settle])
    sw = reps[k]
    return {"switch_t": sw.t, "ring_size": sw.ring_size, "version": sw.version,
            "ms_before": before, "ms_after": after, "switch_ms": cost[k],
            "stall_ms": max(0.0, cost[k] - after),
            "stall_over_step": max(0.0, cost[k] - after) / after}


def elastic_leg_single(args) -> dict:
    """N=1: stop-free scale-out 1 -> 2 workers and scale-in 2 -> 1 on cuda:0 through the
    scheduler-facing API (newcomer prepared on a side thread, switch at Ready + k), aggregate
    batch 512 constant; then stop-resume of the same 1 -> 2 change: checkpoint -> the job is
    torn down -> a FRESH process (new CUDA context, library load, HBM dataset, buffers) loads
    the checkpoint with the new ring and runs its first mini-batch."""
    from paper_1909_11985_b200 import runtime as rt
    settle = 12
    job = rt.Job(_elastic_cfg(512, 1), ["w00"], [0])

    def run(n):
        out = []
        for _ in range(n):
            job.step()
            out.append(job.sync())
        return out

    pre = run(settle + 3)
    t_call = time.perf_counter()
    job.scale_out(["w01"], [0])
    while True:
        r = run(1)[0]
        if r.switched:
            break
        pre.append(r)
    call_to_switch = 1e3 * (time.perf_counter() - t_call)
    reps = pre[-settle:] + [r] + run(settle + 2)
    out = _switch_stall(reps, settle)
    out["call_to_switch_wall_ms"] = call_to_switch
    st = job.scale_in(["w01"])
    pre = run(max(0, st - job.t))
    reps = pre[-settle:] + run(settle + 3)
    sin = _switch_stall(reps, settle)
    from oracle import api, restated  # checker only: the lease log's exactly-once coverage
    ok, _, _ = api.check_coverage(restated(), job.log_text(), WORKLOAD["size"])
    steady = sin["ms_after"]
    # stop-resume: checkpoint, teardown, fresh process, restore, first mini-batch
    import tempfile
    fd, path = tempfile.mkstemp(suffix=".ckpt")
    os.close(fd)
    t0 = time.time()
    job.save_checkpoint(path)
    job.close()
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--_restore", path,
                        "--_ring", "w00,w01"], capture_output=True, text=True, timeout=600)
    child = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    os.unlink(path)
    sr_ms = 1e3 * (child["t_done"] - t0) - steady
    return {"what": "stop-free scale-out 1->2 workers and scale-in 2->1 on one GPU (configs[1] "
                    "MLP, aggregate batch 512, T_a 500 ms) vs stop-resume through a fresh "
                    "process", "scale_out": out, "scale_in": sin,
            "coverage_exactly_once": ok, "stop_resume_ms": sr_ms,
            "stop_resume_parts_ms": child.get("parts_ms"),
            "stall_ms": out["stall_ms"], "stop_resume_over_stall":
                sr_ms / max(out["stall_ms"], 1e-3)}


def restore_child(path: str, ring: str) -> None:
    """--_restore: the resumed job of a stop-resume (fresh process, no torch import)."""
    from paper_1909_11985_b200 import runtime as rt
    t_start = time.time()
    ids = ring.split(",")
    job = rt.Job(_elastic_cfg(512, len(ids)), ids, [0] * len(ids))
    t_built = time.time()
    job.load_checkpoint(path)
    t_loaded = time.time()
    job.step()
    job.sync()
    t_done = time.time()
    print(json.dumps({"t_done": t_done, "parts_ms": {
        "process_start_to_job_built": 1e3 * (t_built - t_start),
        "load_checkpoint": 1e3 * (t_loaded - t_built),
        "first_minibatch": 1e3 * (t_done - t_loaded)}}), flush=True)
    job.close()


def elastic_leg_mp(args, rank: int, world: int, local: int, dist) -> dict:
    """N>1 (one process per GPU): the lower half of the ranks train; the upper half build
    their newcomers with Job.joining while the ring trains and switch in at S1 (the ring copies
    the consolidated model into them over NVLink); at S2 they leave again (scale-in).  Stall =
    switch mini-batch minus the steady mini-batch after it, max over the ring's ranks."""
    from paper_1909_11985_b200 import runtime as rt
    s1, s2, steps = 20, 40, 60
    full = [f"w{r:02d}" for r in range(world)]
    half = world // 2
    ring0, newcomers = full[:half], full[half:]
    cfg = _elastic_cfg(256 * world, world)
    cfg.keep_log = False
    if rank >= half:
        job = rt.Job.joining(cfg, ring0, newcomers, full[rank], local, rank, s1)
    else:
        job = rt.Job(cfg, ring0, [local if r == rank else -1 for r in range(half)])
        job.schedule(s1, True, newcomers, [-1] * len(newcomers))
    job.schedule(s2, False, newcomers)
    blobs = [None] * world
    dist.all_gather_object(blobs, job.export_handles())
    for r, b in enumerate(blobs):
        if r != rank:
            job.import_handles(b)
    dist.barrier()
    ms = {}
    for _ in range(steps):
        rep = job.step()
        if full[rank] not in job.ring():
            if rep.t >= s2:
                break
            continue
        r2 = job.sync()
        ms[rep.t] = r2.step_ms + r2.stall_ms  # incl. the idle gap of the switch's copies
    allms = [None] * world
    dist.all_gather_object(allms, ms)
    dist.barrier()
    job.close()
    per_t = {}
    for m in allms:
        for t, v in m.items():
            per_t[t] = max(per_t.get(t, 0.0), v)

    def stall(s, lo, hi):
        steady = statistics.median(per_t[t] for t in range(lo, hi))
        return {"switch_t": s, "switch_step_ms": per_t[s], "step_ms_after": steady,
                "stall_ms": max(0.0, per_t[s] - steady),
                "stall_over_step": max(0.0, per_t[s] - steady) / steady}

    out = stall(s1, s1 + 3, s2)
    sin = stall(s2, s2 + 3, steps)
    return {"what": f"stop-free scale-out {half}->{world} GPUs and scale-in {world}->{half} "
                    f"across processes (configs[1] MLP, aggregate batch {256 * world})",
            f"scale_out_{half}to{world}": out, f"scale_in_{world}to{half}": sin,
            "stall_ms": out["stall_ms"]}


NCU_FULL = "profiles/r01_ncu_full.md"
NCU_STEP = "profiles/r02f_kernel_shares.md"


def _ncu_traffic(family: str):
    """DRAM read + write bytes per launch of a kernel family: from the round-2 launch list
    with caches not flushed between kernels (profiles/r02f_kernel_shares.md, DRAM table: the
    dirty lines a launch leaves in L2 are counted where they are written back), else the
    round-1 `ncu --set full` capture (profiles/r01_ncu_full.md), or None."""
    here = os.path.dirname(os.path.abspath(__file__))
    try:
        in_dram = False
        for line in open(os.path.join(here, NCU_STEP)):
            in_dram = in_dram or line.startswith("## DRAM traffic")
            cells = [c.strip() for c in line.split("|")]
            if in_dram and len(cells) == 7 and family in cells[1] and cells[2].isdigit():
                return (float(cells[4]) + float(cells[5])) * 1e6 / int(cells[2])
    except (OSError, ValueError):
        pass
    vals = []
    try:
        for line in open(os.path.join(here, NCU_FULL)):
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
    ap.add_argument("--no-elastic", action="store_true",
                    help="skip the stop-free scaling vs stop-resume leg")
    ap.add_argument("--_restore", help=argparse.SUPPRESS)
    ap.add_argument("--_ring", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args._restore:
        restore_child(args._restore, args._ring)
        return
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: launch N ranks of this script (rank 0 prints the line)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_b200(args, rank, world)


if __name__ == "__main__":
    main()
