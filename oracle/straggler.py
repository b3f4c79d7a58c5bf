"""CPU restatement of the straggler rule (test infrastructure only: tests/ may import this).

SPEC.md:348-356 ("its per-mini-batch time is longer than 1.2 times of the
median for 10 mini-batches"): a worker is a straggler if, in each of the last `window`
mini-batches, its duration is strictly greater than `factor` x that mini-batch's median over
the workers present.  The reference has no implementation (spec-only); the restatement fixes
the two choices the spec leaves open exactly as the product does: the median of an even
number of workers is the mean of the two middle values, and with several stragglers the
lowest worker index is returned.  Parity unpinned by reference code (no golden vectors
exist); pinned by the SPEC.md examples in tests/test_straggler.py.
"""
from __future__ import annotations

import math


def detect_straggler(durations, window: int = 10, factor: float = 1.2):
    n_batches = len(durations)
    if window < 1 or n_batches < window or n_batches == 0:
        return None
    n_workers = len(durations[0])
    hits = [0] * n_workers
    for b in range(n_batches - window, n_batches):
        row = durations[b]
        present = sorted(d for d in row if not math.isnan(d))
        if not present:
            return None
        m = len(present)
        med = present[m // 2] if m % 2 else 0.5 * (present[m // 2 - 1] + present[m // 2])
        for k, d in enumerate(row):
            if not math.isnan(d) and d > factor * med:
                hits[k] += 1
    for k in range(n_workers):
        if hits[k] == window:
            return k
    return None
