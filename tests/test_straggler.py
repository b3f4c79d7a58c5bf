"""Straggler detection: the product's rule (C ABI edl_detect_straggler)
against the SPEC examples and the CPU restatement in oracle/straggler.py."""
import math
import random

from oracle.straggler import detect_straggler as oracle_detect
from paper_1909_11985_b200.runtime import detect_straggler


def _matrix(n_batches, n_workers, slow=None, factor=1.0, slow_batches=None, base=100.0):
    rng = random.Random(7)
    rows = []
    for b in range(n_batches):
        row = [base * (1.0 + 0.01 * rng.random()) for _ in range(n_workers)]
        if slow is not None and (slow_batches is None or b >= n_batches - slow_batches):
            row[slow] = base * factor
        rows.append(row)
    return rows


def test_spec_one_worker_at_four_thirds_for_ten_batches_is_flagged():
    # delaying a worker by 1/3 of the mini-batch time; 16 workers
    d = _matrix(12, 16, slow=5, factor=4 / 3)
    assert detect_straggler(d) == 5 == oracle_detect(d)


def test_spec_nine_batches_is_not_enough():
    d = _matrix(12, 16, slow=5, factor=4 / 3, slow_batches=9)
    assert detect_straggler(d) is None and oracle_detect(d) is None


def test_spec_exactly_1_2_times_median_is_not_a_straggler():
    d = [[1.0] * 14 + [1.2, 1.2] for _ in range(10)]
    assert detect_straggler(d) is None and oracle_detect(d) is None


def test_fewer_batches_than_window():
    d = _matrix(9, 4, slow=1, factor=2.0)
    assert detect_straggler(d) is None and oracle_detect(d) is None


def test_absent_workers_and_even_median():
    d = _matrix(10, 4, slow=2, factor=1.5)
    d[3][0] = math.nan  # worker 0 absent from one batch (e.g. joined later)
    assert detect_straggler(d) == 2 == oracle_detect(d)
    two = [[1.0, 1.33] for _ in range(10)]  # median 1.165: 1.33 < 1.2 x 1.165
    assert detect_straggler(two) is None and oracle_detect(two) is None


def test_random_matrices_match_restatement():
    rng = random.Random(3)
    for _ in range(300):
        nb, nw = rng.randint(1, 14), rng.randint(1, 9)
        d = [[rng.choice([1.0, 1.1, 1.25, 1.5, 2.0, math.nan]) for _ in range(nw)]
             for _ in range(nb)]
        w = rng.randint(1, 12)
        f = rng.choice([1.0, 1.2, 1.3])
        assert detect_straggler(d, w, f) == oracle_detect(d, w, f), (d, w, f)
