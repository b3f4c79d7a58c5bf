"""Stall of stop-free scaling vs stop-resume (BASELINE.json configs[2], SPEC.md AC5/AC6).

Single process, one replica per GPU.  The job trains the configs[1] MLP (4096 x 8, bf16)
with a constant aggregate batch B split across the ring and scales
1 -> 2 -> 4 GPUs mid-epoch through Job.scale_out (switch at t + max(1, ceil(T_a / T_b)),
newcomer prepared on a side thread), then 4 -> 2 through Job.scale_in.  For every switch it
reports

  stall_ms      device time of the switch mini-batch above the new steady state (model
                broadcast over NVLink + master consolidation + barrier skew) plus any device
                idle before it
  call_to_switch_wall_ms   scale_out() to the switch: newcomer preparation on the side
                thread (Ready) + k = max(1, ceil(T_a / T_b)) mini-batches

and for scale-out also the stop-resume alternative measured on the same GPUs:
checkpoint (D2H of the fp32 master) -> tear the job down -> build a new job on the larger
GPU set (contexts are warm; datasets, buffers and plans are rebuilt) -> restore -> first
mini-batch, minus one steady-state mini-batch.

  python tools/elastic_bench.py [--gpus 4] [--batch 2048] [--ta 500]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1909_11985_b200 import runtime as rt  # noqa: E402


def cfg_for(args):
    return rt.JobConfig(model=rt.MLP, size=args.size, dim=4096, seed=1, noise=0.0,
                        num_classes=4096, layers=8, hidden=4096, eta=0.05, batch=args.batch,
                        lease_seed=7, partitions=0, max_workers=args.gpus, init_seed=0,
                        t_a_ms=args.ta, keep_log=True)


def run_steps(job, n):
    reps = []
    for _ in range(n):
        job.step()
        reps.append(job.sync())
    return reps


def switch_stats(reps, settle=10):
    """reps: mini-batch reports around one switch (the switch is the first switched one)."""
    k = next(i for i, r in enumerate(reps) if r.switched)
    before = statistics.median(r.step_ms for r in reps[max(0, k - settle):k])
    after = statistics.median(r.step_ms for r in reps[k + 2:k + 2 + settle])
    sw = reps[k]
    return {"t": sw.t, "version": sw.version, "ring_size": sw.ring_size,
            "step_ms_before": before, "step_ms_after": after, "switch_step_ms": sw.step_ms,
            "idle_before_switch_ms": sw.stall_ms,
            "stall_ms": max(0.0, sw.step_ms - after) + sw.stall_ms}


def stop_resume(args, ring_before, devs_before, ring_after, devs_after, warm=20):
    """Checkpoint -> teardown -> rebuild on the new GPU set -> restore -> first step."""
    job = rt.Job(cfg_for(args), ring_before, devs_before)
    run_steps(job, warm)
    t0 = time.perf_counter()
    params = job.params(ring_before[0])
    job.close()
    job = rt.Job(cfg_for(args), ring_after, devs_after)
    job.set_params(params)
    first = run_steps(job, 1)[0]
    t1 = time.perf_counter()
    steady = statistics.median(r.step_ms for r in run_steps(job, 10))
    job.close()
    return {"wall_ms": 1e3 * (t1 - t0), "stall_ms": 1e3 * (t1 - t0) - steady,
            "first_step_ms": first.step_ms, "steady_step_ms": steady}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=4)
    ap.add_argument("--batch", type=int, default=2048, help="aggregate batch B (constant)")
    ap.add_argument("--size", type=int, default=1 << 18, help="dataset samples per GPU")
    ap.add_argument("--ta", type=float, default=500.0, help="switch allowance T_a (ms)")
    ap.add_argument("--settle", type=int, default=30)
    args = ap.parse_args()
    import torch
    ngpu = min(args.gpus, torch.cuda.device_count())
    out = {"workload": "mlp4096x8_bf16", "aggregate_batch": args.batch, "t_a_ms": args.ta,
           "gpus": ngpu, "events": []}

    job = rt.Job(cfg_for(args), ["w00"], [0])
    reps = run_steps(job, args.settle)
    plan = [(["w01"], [1])] if ngpu >= 2 else []
    if ngpu >= 4:
        plan.append((["w02", "w03"], [2, 3]))
    for ids, devs in plan:
        t_call = time.perf_counter()
        t0 = job.t
        job.scale_out(ids, devs)  # newcomers prepared on a side thread from here
        pre = []
        while True:  # switch_t = t_ready + k once the newcomers are Ready
            r = run_steps(job, 1)[0]
            if r.switched:
                break
            pre.append(r)
        prep_wall = 1e3 * (time.perf_counter() - t_call)
        post = [r] + run_steps(job, args.settle + 1)
        stats = switch_stats(pre[-args.settle:] + post, settle=args.settle)
        stats.update({"kind": "scale_out", "ids": ids, "devices": devs,
                      "steps_call_to_switch": r.t - t0, "call_to_switch_wall_ms": prep_wall})
        out["events"].append(stats)
    if ngpu >= 4:
        # straggler replacement (BASELINE configs[3]) at 4 GPUs: w03 slowed by 1/3 of a
        # mini-batch, detected after 10 slow mini-batches (1.2x the median of
        # the four), scaled in, and replaced stop-free by w04 on its GPU
        base = sorted(job.worker_ms("w03")[-10:])[5]
        job.set_worker_delay("w03", 1e3 * base / 3)
        n_slow = 0
        while job.straggler() is None and n_slow < 40:
            run_steps(job, 1)
            n_slow += 1
        t_det = job.t
        w, st, _ = job.replace_straggler("w04", 3)
        pre = []
        while True:
            r = run_steps(job, 1)[0]
            if r.switched:
                break
            pre.append(r)
        post = [r] + run_steps(job, args.settle + 1)
        stats = switch_stats(pre[-args.settle:] + post, settle=args.settle)
        stats.update({"kind": "straggler_replacement", "straggler": w, "replacement": "w04",
                      "slow_minibatches_to_detection": n_slow, "scale_in_switch_t": st,
                      "detected_t": t_det, "ring": job.ring()})
        out["events"].append(stats)
    if ngpu >= 4:
        leave = ["w02", "w04"] if "w04" in job.ring() else ["w02", "w03"]
        st = job.scale_in(leave)
        pre = []
        while job.t < st:
            pre.append(run_steps(job, 1)[0])
        post = run_steps(job, args.settle + 2)
        stats = switch_stats(pre[-args.settle:] + post, settle=args.settle)
        stats.update({"kind": "scale_in", "ids": leave})
        out["events"].append(stats)
    from oracle import api, restated
    ok, fe, detail = api.check_coverage(restated(), job.log_text(), args.size)
    out["coverage_ok"] = ok
    out["ring_final"] = job.ring()
    job.close()

    if ngpu >= 2:
        out["stop_resume_1_to_2"] = stop_resume(args, ["w00"], [0], ["w00", "w01"], [0, 1])
        sf = next(e for e in out["events"] if e["kind"] == "scale_out")
        out["stop_resume_over_stop_free"] = (out["stop_resume_1_to_2"]["stall_ms"] /
                                             max(sf["stall_ms"], 1e-3))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
