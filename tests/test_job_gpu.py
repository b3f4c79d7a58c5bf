"""GPU parity: the product job (libedl_b200.so on a B200) against the reference.

* Linear models (BASELINE.json configs[0], the C1 job): bit-exact against fixtures produced by
  the reference's own ShardManager / SyntheticDataset / accumulate_gradient /
  ring_order_reduce / sgd_step (tests/golden/jobs.json): every per-step loss, every count,
  the final parameters and the assignment log (sha256).
* MLP (configs[1] model family at small width): within tolerance of the numpy oracle
  (oracle/mlp.py) fed with the oracle job driver's lease plan.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def unhex(v):
    return np.array([float.fromhex(x) for x in v], dtype=np.float64)


def run_product(run):
    from paper_1909_11985_b200 import runtime as rt
    spec = run["spec"]
    cfg = rt.JobConfig(model=run["model"], size=spec["size"], dim=spec["dim"], seed=spec["seed"],
                       noise=spec["noise"], sign_labels=spec["sign_labels"], eta=run["eta"],
                       decay=run["decay"], batch=run["B"] or 1,
                       per_worker_batch=run.get("per_worker", 0), lease_seed=run["lease_seed"],
                       partitions=run["d"])
    job = rt.Job(cfg, run["ring"])
    for t, out, ids in run["events"]:
        job.schedule(t, out, ids)
    reps = []
    for _ in range(run["steps"]):
        job.step()
        reps.append(job.sync())
    return job, reps


@pytest.mark.parametrize("name", ["c1_ls", "elastic_mix", "static4_per_worker"])
def test_linear_job_bit_exact(name):
    run = next(r for r in load("jobs.json")["runs"] if r["name"] == name)
    job, reps = run_product(run)
    for rep, (loss_hex, cnt) in zip(reps, run["losses"]):
        assert rep.count == cnt, (rep.t, rep.count, cnt)
        assert float(rep.loss).hex() == loss_hex, (rep.t, rep.loss, float.fromhex(loss_hex))
    w = job.params(job.ring()[0])
    assert np.array_equal(w.view(np.uint64), unhex(run["w_final"]).view(np.uint64))
    text = job.log_text()
    assert hashlib.sha256(text.encode()).hexdigest() == run["log_sha256"]


def test_logistic_job_within_1e12():
    run = next(r for r in load("jobs.json")["runs"] if r["name"] == "c1_logistic")
    job, reps = run_product(run)
    for rep, (loss_hex, cnt) in zip(reps, run["losses"]):
        assert rep.count == cnt
        ref = float.fromhex(loss_hex)
        assert abs(rep.loss - ref) <= 1e-12 * max(1.0, abs(ref))
    w = job.params(job.ring()[0])
    ref = unhex(run["w_final"])
    assert np.max(np.abs(w - ref) / np.maximum(np.abs(ref), 1e-30)) < 1e-9
    assert hashlib.sha256(job.log_text().encode()).hexdigest() == run["log_sha256"]


def test_dataset_f64_bit_exact_and_bf16_rounding():
    import ctypes as C
    from paper_1909_11985_b200 import _lib
    from oracle import mlp as om
    L = _lib.lib()
    for case in load("synthetic_dataset.json")["cases"]:
        spec = case["spec"]
        if spec["size"] * spec["dim"] > (1 << 24):
            continue
        s = _lib.EdlSyntheticSpec(spec["size"], spec["dim"], spec["seed"], spec["noise"],
                                  int(spec["sign_labels"]))
        h = C.c_void_p()
        _lib.check(L.edl_dataset_create_synthetic(C.byref(s), 0, 0, C.byref(h)))
        f = np.zeros(spec["dim"])
        y = C.c_double()
        for smp in case["samples"]:
            _lib.check(L.edl_dataset_get(h, smp["index"], f.ctypes.data_as(C.POINTER(C.c_double)),
                                         C.byref(y)))
            assert hashlib.sha256(f.tobytes()).hexdigest() == smp["features_sha256"]
            assert float(y.value).hex() == smp["label"]
        assert L.edl_dataset_get(h, spec["size"], f.ctypes.data_as(C.POINTER(C.c_double)),
                                 C.byref(y)) == _lib.EDL_OUT_OF_RANGE
        L.edl_dataset_destroy(h)
    # bf16 dataset (MLP workload): f64 -> f32 -> bf16 RNE, int32 class labels
    s = _lib.EdlSyntheticSpec(5000, 96, 3, 0.0, 0)
    h = C.c_void_p()
    _lib.check(L.edl_dataset_create_synthetic(C.byref(s), 1, 40, C.byref(h)))
    ids = np.array([0, 1, 2, 31, 32, 33, 127, 128, 4999], dtype=np.uint64)
    ref = om.features_bf16(3, ids, 96)
    lab = om.labels(3, ids, 40)
    for k, i in enumerate(ids):
        g = np.zeros(96)
        _lib.check(L.edl_dataset_get(h, int(i), g.ctypes.data_as(C.POINTER(C.c_double)), C.byref(y)))
        assert np.array_equal(g.astype(np.float32), ref[k])
        assert int(y.value) == lab[k]
    L.edl_dataset_destroy(h)


def _oracle_plan_steps(spec, B, lease_seed, d, ring, events, steps, per_worker=0):
    from oracle import api, restated
    job = api.Job(restated(), spec, 2, 0.0, 0.0, B, lease_seed, d, ring, per_worker=per_worker)
    for t, out, ids in events:
        job.schedule(t, out, ids)
    plans = []
    for _ in range(steps):
        job.step()
        plans.append([(w, [i for _, i in s]) for w, s in job.plan()])
    return plans, job.log_text()


@pytest.mark.parametrize("momentum", [0.0])
def test_mlp_elastic_vs_numpy_oracle(momentum):
    from oracle.mlp import MLPOracle
    from paper_1909_11985_b200 import runtime as rt
    dim, hidden, classes, layers = 64, 128, 64, 3
    spec = {"size": 3000, "dim": dim, "seed": 5, "noise": 0.0, "sign_labels": False}
    B, steps, eta, decay = 96, 12, 0.1, 0.01
    events = [(4, True, ["w01"]), (9, False, ["w00"])]
    cfg = rt.JobConfig(model=rt.MLP, size=spec["size"], dim=dim, seed=5, noise=0.0,
                       num_classes=classes, layers=layers, hidden=hidden, eta=eta, decay=decay,
                       batch=B, lease_seed=11, partitions=64, init_seed=3, momentum=momentum)
    job = rt.Job(cfg, ["w00"])
    for t, out, ids in events:
        job.schedule(t, out, ids)
    got = []
    for _ in range(steps):
        job.step()
        got.append(job.sync())
    plans, log = _oracle_plan_steps(spec, B, 11, 64, ["w00"], events, steps)
    assert job.log_text() == log  # identical lease plan / membership sequence
    orc = MLPOracle(dim, hidden, classes, layers, 5, 3, eta, decay)
    losses = [orc.step(p, t) for t, p in enumerate(plans)]
    for rep, ref in zip(got, losses):
        assert abs(rep.loss - ref) <= 1e-3 * abs(ref), (rep.t, rep.loss, ref)
    w = job.params(job.ring()[0])
    ref = orc.flat_master()
    w0 = MLPOracle(dim, hidden, classes, layers, 5, 3, eta, decay).flat_master()
    assert np.abs(w - ref).max() <= 1e-3 * np.abs(ref).max()
    assert np.linalg.norm(w - ref) <= 1e-3 * np.linalg.norm(ref)  # north_star: 1e-3 relative
    # the trained change itself agrees (relative error of the total parameter update)
    assert np.linalg.norm((w - w0) - (ref - w0)) <= 2e-2 * np.linalg.norm(ref - w0)


@pytest.mark.parametrize("classes", [4096, 5000])
def test_mlp_wide_softmax_vs_numpy_oracle(classes):
    """Softmax-CE over more than 4096 classes (64 values per thread, BASELINE configs[4] uses
    11264) and the single-member path that reads the loss without a collective launch."""
    from oracle.mlp import MLPOracle
    from paper_1909_11985_b200 import runtime as rt
    dim, hidden, layers, B, steps, eta = 256, 256, 2, 64, 4, 0.1
    spec = {"size": 2000, "dim": dim, "seed": 7, "noise": 0.0, "sign_labels": False}
    cfg = rt.JobConfig(model=rt.MLP, size=spec["size"], dim=dim, seed=7, noise=0.0,
                       num_classes=classes, layers=layers, hidden=hidden, eta=eta, decay=0.0,
                       batch=B, lease_seed=3, partitions=64, init_seed=2)
    job = rt.Job(cfg, ["w00"])
    got = []
    for _ in range(steps):
        job.step()
        got.append(job.sync())
    plans, _ = _oracle_plan_steps(spec, B, 3, 64, ["w00"], [], steps)
    orc = MLPOracle(dim, hidden, classes, layers, 7, 2, eta, 0.0)
    for t, p in enumerate(plans):
        ref = orc.step(p, t)
        assert abs(got[t].loss - ref) <= 1e-3 * abs(ref), (t, got[t].loss, ref)
    w = job.params("w00")
    ref = orc.flat_master()
    w0 = MLPOracle(dim, hidden, classes, layers, 7, 2, eta, 0.0).flat_master()
    err = np.abs(w - ref)
    # bf16 activations / gradients: single-ulp rounding flips between the GPU and numpy are
    # expected, so bound the max by one bf16 ulp of max|w| and the mean tightly (as the
    # multi-GPU parity test does), and require the trained change itself to agree
    assert err.max() <= 2 ** -8 * np.abs(ref).max() and err.mean() <= 1e-4 * np.abs(ref).max()
    assert np.linalg.norm(err) <= 1e-3 * np.linalg.norm(ref)  # north_star: 1e-3 relative
    assert np.linalg.norm((w - w0) - (ref - w0)) <= 2e-2 * np.linalg.norm(ref - w0)


def test_mlp_init_matches_oracle():
    from oracle.mlp import MLPOracle
    from paper_1909_11985_b200 import runtime as rt
    cfg = rt.JobConfig(model=rt.MLP, size=512, dim=64, seed=1, noise=0.0, num_classes=32,
                       layers=2, hidden=96, batch=32, init_seed=9)
    job = rt.Job(cfg, ["w00"])
    orc = MLPOracle(64, 96, 32, 2, 1, 9, 0.1, 0.0)
    assert np.array_equal(job.params("w00"), orc.flat_master())


def test_scale_api_retry_and_k():
    from paper_1909_11985_b200 import runtime as rt
    from paper_1909_11985_b200 import _lib
    cfg = rt.JobConfig(model=rt.LEAST_SQUARES, batch=64, t_a_ms=500.0)
    job = rt.Job(cfg, ["w00"])
    for _ in range(5):
        job.step()
    job.sync()
    # scale_out: the switch is fixed only when the newcomer is Ready
    assert job.scale_out(["w01"]) == -1
    with pytest.raises(_lib.EdlError) as e:
        job.scale_in(["w00"])
    assert e.value.code == _lib.EDL_RETRY
    for _ in range(100000):
        rep = job.step()
        if rep.switched:
            break
    assert rep.switched and rep.ring_size == 2 and rep.version == 2
    job.sync()
    tb = job.median_step_ms()
    st2 = job.scale_in(["w00"])
    assert st2 == job.t + rt.switch_delay(500.0, tb)
    while job.t <= st2:
        job.step()
    job.sync()
    assert job.ring() == ["w01"]
    from oracle import api, restated
    ok, fe, detail = api.check_coverage(restated(), job.log_text(), cfg.size)
    assert ok, detail
