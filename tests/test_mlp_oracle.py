"""CPU: the MLP oracle (oracle/mlp.py) against hand-written statements of the same rules.

The reference has no MLP, so the oracle's update rules are pinned here to
their definitions: plain SGD w -= fp32(eta_t / count) * g (trainer.cpp:56-61), momentum
v = mu*v + g/count, w -= eta_t*v, the fp32 ring-order sum of the members' bf16 gradients,
the bf16 rounding (round to nearest even) and the chunked parallel init.
"""
import numpy as np

from oracle import mlp as om


def _np_bf16(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return r.astype(np.uint32).view(np.float32)


def test_bf16_round_is_rne():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(100000).astype(np.float32) * 10.0 ** rng.integers(-6, 6, 100000)
    ties = np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -(1.0 + 2.0 ** -8)], np.float32)
    for v in (x, ties):
        assert np.array_equal(om.bf16_round(v), _np_bf16(v))


def test_chunked_init_equals_single_pass():
    n_out, n_in = 1100, 4096  # > 2^22 parameters: takes the threaded path
    a = om.init_layer(3, 12345, n_out, n_in)
    b = om._init_chunk(3, 12345, 12345 + n_out * n_in, np.sqrt(6.0 / n_in)).reshape(n_out, n_in)
    assert np.array_equal(a, b)


def _plan(n_workers, ids):
    parts = np.array_split(np.asarray(ids, dtype=np.uint64), n_workers)
    return [(f"w{k:02d}", list(p)) for k, p in enumerate(parts)]


def test_sgd_and_momentum_rules():
    dim, hidden, classes, layers = 32, 48, 16, 3
    eta, decay, mu = 0.3, 0.1, 0.9
    plain = om.MLPOracle(dim, hidden, classes, layers, 2, 5, eta, decay)
    mom = om.MLPOracle(dim, hidden, classes, layers, 2, 5, eta, decay, momentum=mu)
    ref_w = [m.numpy().copy() for m in plain.master]
    ref_m = [m.numpy().copy() for m in mom.master]
    ref_v = [np.zeros_like(m) for m in ref_m]
    rng = np.random.default_rng(1)
    for t in range(4):
        ids = rng.integers(0, 10000, 40)
        plan = _plan(1 + t % 3, ids)
        count = sum(len(i) for _, i in plan)
        # gradients of the members at the current (shared) weights, summed in ring order
        for orc, w in ((plain, ref_w), (mom, ref_m)):
            parts = [orc.worker_grad(np.asarray(i, dtype=np.uint64))[1] for _, i in plan]
            g = [parts[0][l].numpy().copy() for l in range(layers)]
            for p in parts[1:]:
                for l in range(layers):
                    g[l] = (g[l] + p[l].numpy()).astype(np.float32)
            eta_t = eta / (1.0 + decay * t)
            for l in range(layers):
                if orc is plain:
                    w[l] = (w[l] - np.float32(eta_t / count) * g[l]).astype(np.float32)
                else:
                    ref_v[l] = (np.float32(mu) * ref_v[l] + g[l] * np.float32(1.0 / count)
                                ).astype(np.float32)
                    w[l] = (w[l] - np.float32(eta_t) * ref_v[l]).astype(np.float32)
            orc.step(plan, t)
            for l in range(layers):
                assert np.array_equal(orc.master[l].numpy(), w[l]), (t, l)
    assert np.array_equal(mom.flat_mom(), np.concatenate([v.ravel() for v in ref_v]))


def test_worker_grad_matches_float64_within_bf16():
    """The fp32 forward/backward agrees with an f64 evaluation of the same bf16-rounded
    network to bf16 precision on the first (top) layer's gradient."""
    o = om.MLPOracle(64, 64, 32, 2, 4, 1, 0.1, 0.0)
    ids = np.arange(20, dtype=np.uint64)
    loss, g = o.worker_grad(ids)
    W = [om.bf16_round(m.numpy()).astype(np.float64) for m in o.master]
    x = om.features_bf16(4, ids, 64).astype(np.float64)
    y = om.labels(4, ids, 32)
    h = np.maximum(x @ W[0].T, 0.0)
    z = h @ W[1].T
    z = z - z.max(axis=1, keepdims=True)
    p = np.exp(z) / np.exp(z).sum(axis=1, keepdims=True)
    ref_loss = float(-np.log(p[np.arange(20), y]).sum())
    assert abs(loss - ref_loss) <= 1e-3 * abs(ref_loss)
    p[np.arange(20), y] -= 1.0
    g1 = p.T @ h
    assert np.linalg.norm(g[1].numpy() - g1) <= 2e-2 * np.linalg.norm(g1)
