"""Product partition leasing (libedl_b200.so, csrc/lease.cpp) vs the reference ShardManager's
own recorded behaviour (tests/golden/leases.json).  Host-only: runs without a GPU."""
import json
import os

import pytest

from paper_1909_11985_b200 import datapipeline as dp
from paper_1909_11985_b200 import runtime as rt
from paper_1909_11985_b200 import _lib

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def as_tuple(res):
    v = res.value
    if isinstance(v, dp.Shard):
        return ["shard", v.meta.index, v.meta.offset, v.meta.length, v.resume_offset]
    if isinstance(v, dp.EpochEnd):
        return ["epoch_end", v.epoch]
    return ["pending"]


def test_capi_exports_every_header_symbol():
    L = _lib.lib()
    syms = _lib.header_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_permutations_match_reference():
    for p in load("leases.json")["permutations"]:
        sm = dp.ShardManager(p["size"], p["d"], p["seed"], "loc")
        sm.register_worker("w")
        for e, perm in enumerate(p["epoch_perms"]):
            assert sm.permutation() == perm
            for _ in range(p["d"]):
                r = sm.next_shard("w")
                s = r.value
                assert sm.report_progress(dp.ProgressRecord("w", s.meta.index, s.meta.length)) == dp.PipeStatus.Ok
            r = sm.next_shard("w")
            assert r.value == dp.EpochEnd(e)


def test_partition_meta_and_unknown_worker():
    for size, d, p, off, ln in load("leases.json")["partition_meta"]:
        m = dp.ShardManager(size, d, 0).partition_meta(p)
        assert (m.offset, m.length) == (off, ln)
    sm = dp.ShardManager(100, 4, 1)
    assert sm.next_shard("ghost").status == dp.PipeStatus.UnknownWorker
    assert sm.report_progress(dp.ProgressRecord("ghost", 0, 1)) == dp.PipeStatus.UnknownWorker
    sm.register_worker("a")
    assert sm.report_progress(dp.ProgressRecord("a", 0, 1)) == dp.PipeStatus.StaleShard
    assert dp.default_partition_count(2) == 64 and dp.default_partition_count(20) == 80


def replay(s):
    sm = dp.ShardManager(s["size"], s["d"], int(s["seed"]), "x")
    for op, res in zip(s["ops"], s["results"]):
        kind, args = op[0], op[1:]
        got = None
        if kind == "reg":
            sm.register_worker(args[0])
        elif kind == "unreg":
            sm.unregister_worker(args[0])
        elif kind == "next":
            r = sm.next_shard(args[0])
            got = [int(r.status), as_tuple(r) if r.status == dp.PipeStatus.Ok else None]
        elif kind == "report":
            got = int(sm.report_progress(dp.ProgressRecord(*args)))
        elif kind == "reclaim":
            sm.reclaim(args[0])
        elif kind == "reclaim_at":
            sm.reclaim_at(args[0], [tuple(x) for x in args[1]])
        else:
            sm.reclaim_missing(args[0])
        assert got == res, (op, got, res)
    return sm


def test_random_scripts_bit_exact_with_reference():
    for s in load("leases.json")["scripts"]:
        sm = replay(s)
        f = s["final"]
        assert (sm.epoch(), sm.epochs_completed(), sm.cursor(), sm.permutation(),
                sm.reclaimed_count(), sm.in_flight_count()) == (
            f["epoch"], f["epochs_completed"], f["cursor"], f["perm"], f["reclaimed"],
            f["in_flight"])
        assert sm.snapshot().hex() == s["snapshot_hex"]


def test_snapshot_restore_and_errors():
    s = load("leases.json")["scripts"][5]
    sm = replay(s)
    snap = sm.snapshot()
    sm2 = dp.ShardManager(s["size"], s["d"], 0, "other")
    assert sm2.restore(snap) == dp.PipeStatus.Ok
    assert sm2.snapshot() == snap
    assert dp.ShardManager(s["size"] + 1, s["d"], 0).restore(snap) == dp.PipeStatus.ShapeMismatch
    with pytest.raises(_lib.EdlError) as e:
        sm2.restore(snap[:7])
    assert e.value.code == _lib.EDL_ETRUNCATED


def test_scripted_reclaimed_first():
    sm = dp.ShardManager(800, 8, 3)
    sm.register_worker("w0")
    first = sm.next_shard("w0").value
    sm.report_progress(dp.ProgressRecord("w0", first.meta.index, 40))
    sm.register_worker("w1")
    seq = [as_tuple(sm.next_shard("w1"))]
    sm.reclaim("w0")
    sm.unregister_worker("w0")
    seq += [as_tuple(sm.next_shard("w1")), as_tuple(sm.next_shard("w1"))]
    gold = load("leases.json")["scripted"]
    assert [["w0", ["shard", first.meta.index, first.meta.offset, first.meta.length, 0]]] + \
        [["w1", s] for s in seq] == gold


def test_split_batch_and_switch_delay():
    assert rt.split_batch(384, 4) == [96] * 4
    assert rt.split_batch(384, 5) == [77, 77, 77, 77, 76]
    with pytest.raises(_lib.EdlError) as e:
        rt.split_batch(3, 4)
    assert e.value.code == _lib.EDL_EINVAL
    assert rt.switch_delay(500, 250) == 2 and rt.switch_delay(500, 800) == 1
    assert rt.eta_at(0.1, 0.5, 2) == 0.1 / (1 + 0.5 * 2)
