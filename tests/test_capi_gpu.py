"""GPU: the fine-grained C-ABI primitives (include/edl_b200.h) called directly, the way a
reference maintainer's binding would, against the reference's own outputs.

* edl_local_gradient / edl_batch_loss / edl_sgd_step — trainer.cpp:14-61 golden cases
  (tests/golden/trainer.json, generated from the compiled reference) and the SPEC known
  answers (SPEC.md:419 grad [-3,-6]; SPEC.md:428 w' = [0.9]; zero count -> Invalid).
* edl_ring_allreduce_f64 — AC1: the reference's threaded ring_allreduce sums
  for N = 1..8 x len {1, 7, 97, 1024} (tests/golden/collective.json), bit for bit.
* edl_gather — leased runs of sample ids gathered from the HBM dataset equal the
  SyntheticDataset::get rows (dataset.cpp:36-54).
Device buffers come from torch (plumbing only); every computation is the library's kernels.
"""
import ctypes as C
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


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda:0")


def P(t):
    return C.c_void_p(t.data_ptr())


@pytest.fixture(scope="module")
def L():
    import torch
    torch.cuda.set_device(0)
    from paper_1909_11985_b200 import _lib
    return _lib.lib()


def _sync():
    import torch
    torch.cuda.synchronize()


def test_trainer_primitives_match_reference(L):
    import torch
    from paper_1909_11985_b200 import _lib
    g = load("trainer.json")
    for c in g["cases"]:
        n, dim, kind = c["n"], c["dim"], c["model"]
        x = unhex(c["x"]).reshape(n, dim) if n else np.zeros((1, dim))
        y = unhex(c["y"]) if n else np.zeros(1)
        w = dev(unhex(c["w"]))
        xd, yd = dev(x), dev(y)
        grad = torch.full((dim + 1,), float("nan"), dtype=torch.float64, device="cuda:0")
        loss = torch.zeros(1, dtype=torch.float64, device="cuda:0")
        _lib.check(L.edl_local_gradient(kind, P(w), P(xd), P(yd), n, dim, P(grad), None))
        _lib.check(L.edl_batch_loss(kind, P(w), P(xd), P(yd), n, dim, P(loss), None))
        _sync()
        got = grad.cpu().numpy()
        ref = unhex(c["grad"])
        assert got[dim] == n  # the [grad_sum, count] convention, trainer.cpp:244-254
        if kind == 0:  # least squares: bit-exact
            assert np.array_equal(got[:dim].view(np.uint64), ref.view(np.uint64)), c
            assert float(loss.item()).hex() == c["loss"]
        else:  # logistic: CUDA exp/log1p vs glibc (<= 1 ulp)
            assert np.allclose(got[:dim], ref, rtol=1e-12, atol=0)
            assert abs(loss.item() - float.fromhex(c["loss"])) <= 1e-12 * max(1.0, abs(loss.item()))
        if int(c["count"]) == 0:
            continue
        gd = dev(ref if kind == 0 else got[:dim])
        _lib.check(L.edl_sgd_step(P(w), P(gd), int(c["count"]), 0.05, dim, None))
        _sync()
        if kind == 0:
            wa = w.cpu().numpy()
            assert np.array_equal(wa.view(np.uint64), unhex(c["w_after"]).view(np.uint64))


def test_spec_known_answers(L):
    import torch
    from paper_1909_11985_b200 import _lib
    # w=[0,0], one sample a=[1,2], b=3 -> grad = [-3,-6]
    w, x, y = dev([0.0, 0.0]), dev([[1.0, 2.0]]), dev([3.0])
    g = torch.zeros(3, dtype=torch.float64, device="cuda:0")
    _lib.check(L.edl_local_gradient(0, P(w), P(x), P(y), 1, 2, P(g), None))
    _sync()
    assert g.cpu().tolist() == [-3.0, -6.0, 1.0]
    # empty batch -> ([0, 0], 0)
    _lib.check(L.edl_local_gradient(0, P(w), P(x), P(y), 0, 2, P(g), None))
    _sync()
    assert g.cpu().tolist() == [0.0, 0.0, 0.0]
    # w=[1], grad_sum=[2], count=2, eta=0.1 -> [0.9]; grad 0 -> fixed point
    w1, g1 = dev([1.0]), dev([2.0, 2.0])
    _lib.check(L.edl_sgd_step(P(w1), P(g1), 2, 0.1, 1, None))
    _sync()
    assert float(w1.item()).hex() == load("trainer.json")["spec_sgd"][0]
    # count read from the device slot g[dim] (count < 0)
    w2 = dev([1.0])
    _lib.check(L.edl_sgd_step(P(w2), P(g1), -1, 0.1, 1, None))
    _sync()
    assert w2.item() == w1.item()
    z = dev([0.0, 0.0])
    _lib.check(L.edl_sgd_step(P(w2), P(z), 5, 0.1, 1, None))
    _sync()
    assert w2.item() == w1.item()
    # zero count -> Invalid (trainer.cpp:57-58 throws invalid_argument)
    assert L.edl_sgd_step(P(w2), P(g1), 0, 0.1, 1, None) == _lib.EDL_EINVAL
    assert L.edl_local_gradient(0, P(w), P(x), P(y), 1, 0, P(g), None) == _lib.EDL_EINVAL


def test_ring_allreduce_f64_matches_reference_collective(L):
    """AC1: the kernel's chunk-ordered sum equals the reference's threaded ring_allreduce."""
    import torch
    from oracle.gen_golden import det_vector
    from paper_1909_11985_b200 import _lib
    for c in load("collective.json")["cases"]:
        n, ln = c["n"], c["len"]
        ins = [dev(det_vector(c["seed_base"] + r, ln)) for r in range(n)]
        ptrs = (C.c_void_p * n)(*[t.data_ptr() for t in ins])
        out = torch.empty(ln, dtype=torch.float64, device="cuda:0")
        _lib.check(L.edl_ring_allreduce_f64(ptrs, n, ln, 0, P(out), None))
        _sync()
        got = out.cpu().numpy()
        assert hashlib.sha256(got.tobytes()).hexdigest() == c["sum_sha256"], (n, ln)
        assert float(got[0]).hex() == c["head"][0]
        # Average = Sum / n elementwise (ReduceOp::Average, allreduce.cpp:124-127)
        _lib.check(L.edl_ring_allreduce_f64(ptrs, n, ln, 1, P(out), None))
        _sync()
        assert np.array_equal(out.cpu().numpy(), got / n)
    assert L.edl_ring_allreduce_f64(ptrs, 0, 4, 0, P(out), None) == _lib.EDL_EINVAL


@pytest.mark.parametrize("dtype", [0, 1])
def test_gather_rows_equal_dataset_get(L, dtype):
    import torch
    from paper_1909_11985_b200 import _lib
    dim, size, classes = 96, 5000, 40
    s = _lib.EdlSyntheticSpec(size, dim, 3, 0.01, 0)
    h = C.c_void_p()
    _lib.check(L.edl_dataset_create_synthetic(C.byref(s), dtype, classes, C.byref(h)))
    # ragged leased runs, crossing partition-like boundaries, the last sample included
    runs_py = [(17, 5), (4990, 10), (0, 1), (2048, 33), (1000, 0), (311, 7)]
    n = sum(c for _, c in runs_py)
    runs = (_lib.EdlRun * len(runs_py))(*[_lib.EdlRun(a, c) for a, c in runs_py])
    runs_dev = torch.tensor([v for r in runs_py for v in r], dtype=torch.int64, device="cuda:0")
    xt = torch.bfloat16 if dtype == 1 else torch.float64
    yt = torch.int32 if dtype == 1 else torch.float64
    x = torch.empty((n, dim), dtype=xt, device="cuda:0")
    y = torch.empty(n, dtype=yt, device="cuda:0")
    _lib.check(L.edl_gather(h, C.c_void_p(runs_dev.data_ptr()), len(runs_py), n, P(x), P(y),
                            None))
    _sync()
    xs, ys = x.float().cpu().numpy() if dtype == 1 else x.cpu().numpy(), y.cpu().numpy()
    row = 0
    f = np.zeros(dim)
    lab = C.c_double()
    for a, c in runs_py:
        for i in range(a, a + c):
            _lib.check(L.edl_dataset_get(h, i, f.ctypes.data_as(C.POINTER(C.c_double)),
                                         C.byref(lab)))
            if dtype == 1:
                assert np.array_equal(xs[row], f.astype(np.float32)), i
                assert int(ys[row]) == int(lab.value)
            else:
                assert np.array_equal(xs[row].view(np.uint64), f.view(np.uint64)), i
                assert float(ys[row]).hex() == float(lab.value).hex()
            row += 1
    del runs
    L.edl_dataset_destroy(h)
