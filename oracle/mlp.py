"""ORACLE — TEST INFRASTRUCTURE ONLY.

CPU restatement of the MLP SGD step that BASELINE.json configs[1] / configs[4] ask for.  The
reference has no MLP (linear models only), so this oracle restates the
reference's SGD semantics — grad_sum over the batch, global count, w -= (eta_t / count) * g
(src/trainer.cpp:56-61, applied as trainer.cpp:244-271; eta_at trainer.hpp:27-29) — for a
ReLU MLP with softmax cross-entropy, with the same rounding points as the GPU path:

  features bf16 (f64 -> f32 -> bf16 RNE), weights bf16 working copy of an fp32 master,
  GEMMs accumulate in fp32, hidden activations / dgrads / weight grads rounded to bf16,
  logits fp32, update in fp32 with separate multiply and subtract roundings.

Momentum (north_star "SGD/momentum"; the reference has none) follows the heavy-ball form the
GPU's update kernels use: v = mu*v + g/count, w -= eta_t*v (fp32, every product and sum
rounded separately), v starting at zero.

Integer work (splitmix64 features / labels / init) is numpy uint64; floating point runs in
torch CPU fp32 (multi-threaded BLAS, bf16 rounding via torch's RNE cast) so the oracle covers
the full-size configs in seconds per step.  Parity against it is "within tolerance" (fp32
accumulation order differs), not bit-exact: DESIGN.md §6 states the tolerances.  Used by
tests/, __graft_entry__.smoke() and bench.py's CPU leg only.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

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


def bf16_round_t(x: torch.Tensor) -> torch.Tensor:
    """fp32 -> bf16 round-to-nearest-even, returned as fp32 values (torch CPU)."""
    return x.to(torch.bfloat16).to(torch.float32)


def bf16_round(x) -> np.ndarray:
    """numpy face of bf16_round_t."""
    return bf16_round_t(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))).numpy()


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


def _init_chunk(seed: int, lo: int, hi: int, bound: float) -> np.ndarray:
    idx = np.arange(lo, hi, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) ^ (idx * GOLD + INIT_ADD))
    return ((2.0 * unit(h) - 1.0) * bound).astype(np.float32)


def init_layer(seed: int, offset: int, n_out: int, n_in: int) -> np.ndarray:
    """fp32 master of one layer: float((2u - 1) * sqrt(6 / fan_in)), u from splitmix64 of the
    global parameter index (chunked over threads: numpy ufuncs release the GIL)."""
    n = n_out * n_in
    bound = np.sqrt(6.0 / n_in)
    step = 1 << 22
    if n <= step:
        return _init_chunk(seed, offset, offset + n, bound).reshape(n_out, n_in)
    out = np.empty(n, dtype=np.float32)
    cuts = list(range(0, n, step)) + [n]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        futs = [(a, ex.submit(_init_chunk, seed, offset + a, offset + b, bound))
                for a, b in zip(cuts[:-1], cuts[1:])]
        for a, f in futs:
            v = f.result()
            out[a:a + len(v)] = v
    return out.reshape(n_out, n_in)


class MLPOracle:
    def __init__(self, dim, hidden, classes, layers, data_seed, init_seed, eta, decay,
                 momentum=0.0):
        self.shapes = []
        off = 0
        self.master = []
        for l in range(layers):
            n_in = dim if l == 0 else hidden
            n_out = classes if l == layers - 1 else hidden
            self.shapes.append((n_out, n_in, off))
            self.master.append(torch.from_numpy(init_layer(init_seed, off, n_out, n_in)))
            off += n_out * n_in
        self.dim, self.classes, self.data_seed = dim, classes, data_seed
        self.eta, self.decay, self.momentum = eta, decay, float(momentum)
        self.mom = [torch.zeros_like(m) for m in self.master] if self.momentum else None

    def flat_master(self) -> np.ndarray:
        return torch.cat([m.reshape(-1) for m in self.master]).numpy()

    def flat_mom(self) -> np.ndarray:
        if self.mom is None:
            return np.zeros(sum(m.numel() for m in self.master), dtype=np.float32)
        return torch.cat([v.reshape(-1) for v in self.mom]).numpy()

    def set_state(self, master: np.ndarray, mom: np.ndarray | None = None):
        """Load a flat fp32 master (+ momentum) — e.g. a checkpoint restored mid-run."""
        at = 0
        for l, (n_out, n_in, _) in enumerate(self.shapes):
            n = n_out * n_in
            self.master[l] = torch.from_numpy(
                np.array(master[at:at + n], dtype=np.float32).reshape(n_out, n_in))
            if self.mom is not None and mom is not None:
                self.mom[l] = torch.from_numpy(
                    np.array(mom[at:at + n], dtype=np.float32).reshape(n_out, n_in))
            at += n

    def worker_grad(self, ids, W=None):
        """(loss_sum, [bf16 dW per layer as fp32 tensors]) for one worker's batch."""
        L = len(self.master)
        if W is None:
            W = [bf16_round_t(m) for m in self.master]
        n = len(ids)
        if n == 0:
            return 0.0, [torch.zeros_like(m) for m in self.master]
        x = torch.from_numpy(features_bf16(self.data_seed, ids, self.dim))
        y = torch.from_numpy(labels(self.data_seed, ids, self.classes))
        acts = [x]
        logits = None
        for l in range(L):
            z = acts[-1] @ W[l].T
            if l < L - 1:
                acts.append(bf16_round_t(torch.clamp_min(z, 0.0)))
            else:
                logits = z
        rows = torch.arange(n)
        m = logits.max(dim=1, keepdim=True).values
        e = torch.exp(logits - m)
        s = e.sum(dim=1, keepdim=True)
        p = e / s
        row_loss = (torch.log(s[:, 0]) + m[:, 0] - logits[rows, y]).to(torch.float64)
        p[rows, y] -= 1.0
        dy = bf16_round_t(p)
        grads = [None] * L
        for l in range(L - 1, -1, -1):
            grads[l] = bf16_round_t(dy.T @ acts[l])
            if l > 0:
                dy = bf16_round_t((dy @ W[l]) * (acts[l] > 0))
        return float(row_loss.sum()), grads

    def step(self, plan, t):
        """plan: [(worker, [ids...]), ...] in ring order.  Returns mean loss."""
        count = sum(len(ids) for _, ids in plan)
        W = [bf16_round_t(m) for m in self.master]
        loss = 0.0
        g = None
        for _, ids in plan:  # ring order: fp32 sum of the members' bf16 gradients
            ls, gr = self.worker_grad(np.asarray(ids, dtype=np.uint64), W)
            loss += ls
            g = gr if g is None else [a + b for a, b in zip(g, gr)]
        if count:
            eta_t = self.eta / (1.0 + self.decay * t)
            for l in range(len(self.master)):
                if self.mom is not None:
                    inv = torch.tensor(1.0 / count, dtype=torch.float32)
                    v = self.momentum_f32() * self.mom[l] + g[l] * inv
                    self.mom[l] = v
                    self.master[l] = self.master[l] - torch.tensor(eta_t, dtype=torch.float32) * v
                else:
                    scale = torch.tensor(eta_t / count, dtype=torch.float32)
                    self.master[l] = self.master[l] - scale * g[l]
        return loss / count if count else 0.0

    def momentum_f32(self) -> torch.Tensor:
        return torch.tensor(self.momentum, dtype=torch.float32)
