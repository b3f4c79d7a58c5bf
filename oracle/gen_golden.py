"""ORACLE — TEST INFRASTRUCTURE ONLY.

Generates tests/golden/*.json from the REFERENCE itself (oracle/_ref/libedlref.so, compiled
from /root/reference/proj/src by `make -C oracle ref`).  Run in this container:

    python -m oracle.gen_golden

Floats are stored with float.hex() so fixtures are bit-exact.  The fixtures travel with the
repo; /root/reference does not (nothing on the GPU box reads it).
"""
from __future__ import annotations

import hashlib
import json
import os
import random

import numpy as np

from . import build, reference
from . import api

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
M64 = (1 << 64) - 1


def sm64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def det_vector(seed: int, n: int) -> list[float]:
    """Deterministic f64 inputs in [-1, 1) for collective fixtures."""
    out, s = [], seed
    for _ in range(n):
        s = sm64(s)
        out.append(2.0 * ((s >> 11) * 2.0 ** -53) - 1.0)
    return out


def hx(a) -> list[str]:
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def dump(name: str, obj) -> None:
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, indent=1, sort_keys=True)
    print("wrote", name)


def gen_synth(R):
    specs = [
        {"size": 1000, "dim": 4, "seed": 7, "noise": 0.0, "sign_labels": False},
        {"size": 8192, "dim": 64, "seed": 1, "noise": 0.01, "sign_labels": False},
        {"size": 8192, "dim": 64, "seed": 1, "noise": 0.0, "sign_labels": True},
        {"size": 1000, "dim": 4096, "seed": 9, "noise": 0.0, "sign_labels": True},
        {"size": 300, "dim": 7, "seed": 123456789, "noise": 0.5, "sign_labels": False},
        {"size": 1 << 20, "dim": 4096, "seed": 1, "noise": 0.0, "sign_labels": False},
    ]
    cases = []
    for spec in specs:
        idx = sorted({0, 1, 3, 7, spec["size"] // 2, spec["size"] - 1})
        samples = []
        for i in idx:
            rc, f, y = api.synth_get(R, spec, i)
            assert rc == 0
            samples.append({"index": i, "features": hx(f) if spec["dim"] <= 64 else hx(f[:16]) + hx(f[-16:]),
                            "features_sha256": hashlib.sha256(f.tobytes()).hexdigest(),
                            "label": float(y).hex()})
        rc, _, _ = api.synth_get(R, spec, spec["size"])
        cases.append({"spec": spec, "true_weights_sha256":
                      hashlib.sha256(api.true_weights(R, spec).tobytes()).hexdigest(),
                      "true_weights_head": hx(api.true_weights(R, spec)[:8]),
                      "samples": samples, "out_of_range_rc": rc})
    dump("synthetic_dataset.json", {"source": "reference SyntheticDataset (dataset.cpp:27-54)",
                                    "cases": cases})


def gen_leases(R):
    out = {"source": "reference ShardManager (datapipeline.cpp)"}
    perms = []
    for size, d, seed in [(1000, 64, 0), (1000, 8, 42), (8192, 64, 7), (1 << 20, 64, 7), (100, 4, 5)]:
        lm = api.Leases(R, size, d, seed, "loc")
        lm.register("w")
        epochs = []
        for e in range(3):
            epochs.append(lm.permutation())
            for _ in range(d):
                st, v = lm.next("w")
                assert v[0] == "shard"
                lm.report("w", v[1], v[3])
            st, v = lm.next("w")
            assert v[0] == "epoch_end" and v[1] == e
        perms.append({"size": size, "d": d, "seed": seed, "epoch_perms": epochs})
    out["permutations"] = perms
    lm = api.Leases(R, 8192, 64, 7)
    lm2 = api.Leases(R, 1000, 64, 7)
    out["partition_meta"] = [[8192, 64, p, *lm.meta(p)] for p in (0, 5, 63)] + \
                            [[1000, 64, p, *lm2.meta(p)] for p in (0, 5, 62, 63)]
    # SURVEY Appendix A scripted reclaimed-first sequence
    lm = api.Leases(R, 800, 8, 3)
    seq = []
    lm.register("w0")
    seq.append(("w0", lm.next("w0")[1]))
    p0 = seq[-1][1][1]
    lm.report("w0", p0, 40)
    lm.register("w1")
    seq.append(("w1", lm.next("w1")[1]))
    lm.reclaim("w0")
    lm.unregister("w0")
    seq.append(("w1", lm.next("w1")[1]))
    seq.append(("w1", lm.next("w1")[1]))
    out["scripted"] = [[w, list(v)] for w, v in seq]
    # random scripts: op stream + every return value + final state
    scripts = []
    rng = random.Random(2024)
    for s in range(60):
        size = rng.randint(1, 5000)
        d = rng.randint(1, 70)
        seed = rng.getrandbits(64)
        workers = [f"w{i}" for i in range(5)]
        lm = api.Leases(R, size, d, seed, "x")
        ops, results = [], []
        for _ in range(400):
            w = rng.choice(workers)
            op = rng.choice(["reg", "reg", "next", "next", "next", "report", "report", "reclaim",
                             "unreg", "reclaim_at", "missing"])
            if op == "reg":
                lm.register(w); res = None; args = [w]
            elif op == "unreg":
                lm.unregister(w); res = None; args = [w]
            elif op == "next":
                st, v = lm.next(w); res = [st, list(v) if v else None]; args = [w]
            elif op == "report":
                shards = lm.worker_shards(w)
                if shards and rng.random() < 0.8:
                    p, off = rng.choice(shards)
                    _, ln = lm.meta(p)
                    noff = min(ln, off + rng.randint(0, max(1, ln)))
                else:
                    p, noff = rng.randint(0, d - 1), rng.randint(0, 50)
                res = lm.report(w, p, noff); args = [w, p, noff]
            elif op == "reclaim":
                lm.reclaim(w); res = None; args = [w]
            elif op == "reclaim_at":
                shards = lm.worker_shards(w)
                pairs = [(p, max(0, off - rng.randint(0, 3))) for p, off in shards]
                lm.reclaim_at(w, pairs); res = None; args = [w, pairs]
            else:
                live = [x for x in workers if rng.random() < 0.7]
                lm.reclaim_missing(live); res = None; args = [live]
            ops.append([op] + [a if not isinstance(a, list) else a for a in args])
            results.append(res)
        scripts.append({"size": size, "d": d, "seed": str(seed), "ops": ops, "results": results,
                        "final": {"epoch": lm.epoch(), "epochs_completed": lm.epochs_completed(),
                                  "cursor": lm.cursor(), "perm": lm.permutation(),
                                  "reclaimed": lm.reclaimed_count(),
                                  "in_flight": lm.in_flight_count()},
                        "snapshot_hex": lm.snapshot().hex()})
    out["scripts"] = scripts
    dump("leases.json", out)


def gen_trainer(R):
    cases = []
    rng = np.random.default_rng(11)
    for model in (0, 1):
        for n, dim in [(0, 3), (1, 2), (5, 7), (64, 64), (33, 129)]:
            x = rng.uniform(-1, 1, size=(n, dim))
            y = rng.uniform(-2, 2, size=n) if model == 0 else np.sign(rng.uniform(-1, 1, size=n))
            w = rng.uniform(-1, 1, size=dim)
            g = np.zeros(dim)
            R.local_gradient(model, api._dp(w), dim, api._dp(np.ascontiguousarray(x)),
                             api._dp(y), n, api._dp(g))
            loss = R.batch_loss(model, api._dp(w), dim, api._dp(np.ascontiguousarray(x)),
                                api._dp(y), n)
            w2 = w.copy()
            cnt = max(n, 1)
            R.sgd_step(api._dp(w2), api._dp(g), dim, cnt, 0.05)
            cases.append({"model": model, "n": n, "dim": dim, "x": hx(x), "y": hx(y), "w": hx(w),
                          "grad": hx(g), "loss": float(loss).hex(), "count": cnt,
                          "w_after": hx(w2)})
    # SPEC known answers
    z = np.zeros(2)
    g = np.zeros(2)
    R.local_gradient(0, api._dp(z), 2, api._dp(np.array([1.0, 2.0])), api._dp(np.array([3.0])),
                     1, api._dp(g))
    w1 = np.array([1.0])
    R.sgd_step(api._dp(w1), api._dp(np.array([2.0])), 1, 2, 0.1)
    zero_rc = R.sgd_step(api._dp(w1.copy()), api._dp(np.array([2.0])), 1, 0, 0.1)
    dump("trainer.json", {"source": "reference trainer.cpp:14-61", "cases": cases,
                          "spec_local_gradient": hx(g), "spec_sgd": hx(w1),
                          "zero_count_rc": zero_rc})


def gen_collective(R):
    cases = []
    for n in range(1, 9):
        for ln in (1, 7, 97, 1024):
            inp = np.array([det_vector(1000 * n + ln + r, ln) for r in range(n)])
            out_threads = np.zeros(n * ln)
            transfers = R.ring_allreduce_threads(api._dp(inp), n, ln, api._dp(out_threads))
            order = api.ring_reduce(R, inp)
            per_rank = out_threads.reshape(n, ln)
            assert transfers == 2 * (n - 1) or n == 1, transfers
            assert all(np.array_equal(per_rank[r].view(np.uint64), order.view(np.uint64))
                       for r in range(n)), (n, ln)
            cases.append({"n": n, "len": ln, "seed_base": 1000 * n + ln,
                          "transfers": transfers, "sum_sha256": hashlib.sha256(order.tobytes()).hexdigest(),
                          "head": hx(order[:4])})
    dump("collective.json", {"source": "reference ring_allreduce over InProcFabric threads == "
                                       "ring_order_reduce (allreduce.cpp:60-148)", "cases": cases})


def gen_jobs(R):
    runs = []
    scenarios = [
        # C1: reference default synthetic SGD job, 1 -> 2 workers, stop-free scale-out at t=50
        {"name": "c1_ls", "spec": {"size": 8192, "dim": 64, "seed": 1, "noise": 0.01,
                                    "sign_labels": False},
         "model": 0, "eta": 0.05, "decay": 0.0, "B": 64, "lease_seed": 7, "d": 64,
         "ring": ["w00"], "events": [[50, True, ["w01"]]], "steps": 300},
        {"name": "c1_logistic", "spec": {"size": 8192, "dim": 64, "seed": 1, "noise": 0.0,
                                          "sign_labels": True},
         "model": 1, "eta": 0.5, "decay": 0.01, "B": 64, "lease_seed": 7, "d": 64,
         "ring": ["w00"], "events": [[50, True, ["w01"]]], "steps": 300},
        # C3/C4-style protocol: out 1->2->4, in 4->3 (leaver mid-shard), uneven splits,
        # epoch tails with ShardPending
        {"name": "elastic_mix", "spec": {"size": 1000, "dim": 16, "seed": 3, "noise": 0.1,
                                          "sign_labels": False},
         "model": 0, "eta": 0.02, "decay": 0.001, "B": 96, "lease_seed": 11, "d": 64,
         "ring": ["w00"], "events": [[10, True, ["w01"]], [25, True, ["w03", "w02"]],
                                     [40, False, ["w01"]], [60, True, ["w05"]],
                                     [70, False, ["w00", "w03"]]], "steps": 90},
        {"name": "static4_per_worker", "spec": {"size": 4096, "dim": 32, "seed": 5, "noise": 0.0,
                                                 "sign_labels": False},
         "model": 0, "eta": 0.01, "decay": 0.0, "B": 0, "per_worker": 100, "lease_seed": 9,
         "d": 64, "ring": ["w00", "w01", "w02", "w03"], "events": [], "steps": 40},
    ]
    for sc in scenarios:
        job = api.Job(R, sc["spec"], sc["model"], sc["eta"], sc["decay"], sc["B"],
                      sc["lease_seed"], sc["d"], sc["ring"], per_worker=sc.get("per_worker", 0))
        for t, out, ids in sc["events"]:
            job.schedule(t, out, ids)
        losses = []
        for _ in range(sc["steps"]):
            loss, cnt = job.step()
            losses.append([float(loss).hex(), cnt])
        w = job.params()
        text = job.log_text()
        ok, fe, detail = api.check_coverage(R, text, sc["spec"]["size"])
        rok, rw, rb, rerr = api.replay(R, text, sc["model"], sc["spec"], np.zeros(sc["spec"]["dim"]),
                                       sc["eta"], sc["decay"], True)
        cok, cw, _, _ = api.replay(R, text, sc["model"], sc["spec"], np.zeros(sc["spec"]["dim"]),
                                   sc["eta"], sc["decay"], False)
        assert ok and rok and cok, (sc["name"], detail, rerr)
        runs.append({**sc, "losses": losses, "w_final": hx(w),
                     "log_sha256": hashlib.sha256(text.encode()).hexdigest(),
                     "log_head": text.splitlines()[:6], "log_records": len(text.splitlines()),
                     "coverage_full_epochs": fe,
                     "replay_ring_bit_exact": bool(np.array_equal(rw.view(np.uint64), w.view(np.uint64))),
                     "replay_concat_maxrel": float(np.max(np.abs(cw - w) / np.maximum(
                         np.maximum(np.abs(cw), np.abs(w)), 1e-30)))})
        print(sc["name"], "loss0", float.fromhex(losses[0][0]), "lossN",
              float.fromhex(losses[-1][0]), "epochs", fe, "records", runs[-1]["log_records"])
    with open(os.path.join(OUT, "c1_ls_assignment.log"), "w") as f:
        job = api.Job(R, scenarios[0]["spec"], 0, 0.05, 0.0, 64, 7, 64, ["w00"])
        job.schedule(50, True, ["w01"])
        for _ in range(300):
            job.step()
        f.write(job.log_text())
    dump("jobs.json", {"source": "oracle/job_driver.hpp protocol over reference ShardManager, "
                                  "SyntheticDataset, accumulate_gradient, ring_order_reduce, "
                                  "sgd_step; audited by reference check_coverage/oracle_replay",
                       "runs": runs})


def main():
    build(ref=True)
    R = reference()
    assert R is not None, "oracle/_ref/libedlref.so not built (needs /root/reference)"
    gen_synth(R)
    gen_leases(R)
    gen_trainer(R)
    gen_collective(R)
    gen_jobs(R)


if __name__ == "__main__":
    main()
