"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy restatement of the MLP SGD step that BASELINE.json configs[1] asks for.  The reference
has no MLP (linear models only), so this oracle restates the reference's SGD
semantics — grad_sum over the batch, global count, w -= (eta_t / count) * g
(src/trainer.cpp:56-61, applied as trainer.cpp:244-271; eta_at trainer.hpp:27-29) — for a
ReLU MLP with softmax cross-entropy, with the same rounding points as the GPU path:

  features bf16 (f64 -> f32 -> bf16 RNE), weights bf16 working copy of an fp32 master,
  GEMMs accumulate in fp32, hidden activations / dgrads / weight grads rounded to bf16,
  logits fp32, update in fp32 with separate multiply and subtract roundings.

Parity against it is therefore "within tolerance" (fp32 accumulation order differs), not
bit-exact: DESIGN.md §5 states the tolerances.  Used by tests/ and bench.py's CPU leg only.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLD = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
IDX_MUL = np.uint64(0xD1342543DE82EF95)
INIT_ADD = np.uint64(0x632BE59BD9B4E019)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """src/dataset.cpp:13-18, vectorised over uint64 arrays (wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        x = x + GOLD
        x = (x ^ (x >> np.uint64(30))) * C1
        x = (x ^ (x >> np.uint64(27))) * C2
        return x ^ (x >> np.uint64(31))


def unit(bits: np.ndarray) -> np.ndarray:  # dataset.cpp:20-23
    return (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def bf16_round(x: np.ndarray) -> np.ndarray:
    """f32 -> bf16 round-to-nearest-even, returned as f32 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000))
    return r.astype(np.uint32).view(np.float32)


def features_bf16(seed: int, ids: np.ndarray, dim: int) -> np.ndarray:
    """SyntheticDataset::get features (dataset.cpp:41-47) rounded f64 -> f32 -> bf16."""
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = splitmix64(np.uint64(seed) ^ (ids * IDX_MUL + np.uint64(1)))
    out = np.empty((len(ids), dim), dtype=np.float32)
    for k in range(dim):
        st = splitmix64(st)
        out[:, k] = (2.0 * unit(st) - 1.0).astype(np.float32)
    return bf16_round(out)


def labels(seed: int, ids: np.ndarray, classes: int) -> np.ndarray:
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        st = splitmix64(np.uint64(seed) ^ ~(ids * IDX_MUL + np.uint64(1)))
    return (st % np.uint64(classes)).astype(np.int64)


def init_layer(seed: int, offset: int, n_out: int, n_in: int) -> np.ndarray:
    """fp32 master of one layer: float((2u - 1) * sqrt(6 / fan_in))."""
    idx = np.arange(offset, offset + n_out * n_in, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) ^ (idx * GOLD + INIT_ADD))
    bound = np.sqrt(6.0 / n_in)
    return ((2.0 * unit(h) - 1.0) * bound).astype(np.float32).reshape(n_out, n_in)


class MLPOracle:
    def __init__(self, dim, hidden, classes, layers, data_seed, init_seed, eta, decay):
        self.shapes = []
        off = 0
        self.master = []
        for l in range(layers):
            n_in = dim if l == 0 else hidden
            n_out = classes if l == layers - 1 else hidden
            self.shapes.append((n_out, n_in, off))
            self.master.append(init_layer(init_seed, off, n_out, n_in))
            off += n_out * n_in
        self.dim, self.classes, self.data_seed = dim, classes, data_seed
        self.eta, self.decay = eta, decay

    def flat_master(self) -> np.ndarray:
        return np.concatenate([m.ravel() for m in self.master])

    def worker_grad(self, ids):
        """(loss_sum, [bf16 dW per layer]) for one worker's batch."""
        L = len(self.master)
        W = [bf16_round(m) for m in self.master]
        n = len(ids)
        if n == 0:
            return 0.0, [np.zeros_like(m) for m in self.master]
        x = features_bf16(self.data_seed, ids, self.dim)
        y = labels(self.data_seed, ids, self.classes)
        acts = [x]
        for l in range(L):
            z = acts[-1] @ W[l].T
            if l < L - 1:
                acts.append(bf16_round(np.maximum(z, 0.0)))
            else:
                logits = z.astype(np.float32)
        m = logits.max(axis=1, keepdims=True)
        e = np.exp(logits - m)
        s = e.sum(axis=1, keepdims=True)
        p = e / s
        row_loss = (np.log(s[:, 0]) + m[:, 0] - logits[np.arange(n), y]).astype(np.float64)
        p[np.arange(n), y] -= 1.0
        dy = bf16_round(p)
        grads = [None] * L
        for l in range(L - 1, -1, -1):
            grads[l] = bf16_round(dy.T @ acts[l])
            if l > 0:
                dy = bf16_round((dy @ W[l]) * (acts[l] > 0))
        return float(row_loss.sum()), grads

    def step(self, plan, t):
        """plan: [(worker, [ids...]), ...] in ring order.  Returns mean loss."""
        count = sum(len(ids) for _, ids in plan)
        parts = [self.worker_grad(np.asarray(ids, dtype=np.uint64)) for _, ids in plan]
        loss = 0.0
        for ls, _ in parts:
            loss += ls
        if count:
            eta_t = self.eta / (1.0 + self.decay * t)
            scale = np.float32(eta_t / count)
            for l in range(len(self.master)):
                g = parts[0][1][l].astype(np.float32)
                for _, gr in parts[1:]:
                    g = (g + gr[l]).astype(np.float32)
                self.master[l] = (self.master[l] - (scale * g).astype(np.float32)).astype(np.float32)
        return loss / count if count else 0.0
