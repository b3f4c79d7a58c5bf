"""Leader election with leases (the reference's LeaseStore,
coordination.cpp:26-117), as paper_1909_11985_b200/control.py's LeaderLease runs it on a
torch.distributed Store: the SPEC's examples, the uniqueness / generation-monotonicity
properties under random interleavings on an injectable clock, and a 4-process election over
the rendezvous TCPStore (gloo, CPU) with a graceful handoff."""
import random
import socket
import threading

import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_11985_b200.control import LeaderLease, ManualClock

WON, LOST, OK, NOT = LeaderLease.WON, LeaderLease.LOST, LeaderLease.OK, LeaderLease.NOT_LEADER


def lease(ttl=3.0):
    clk = ManualClock(100.0)
    return LeaderLease(dist.HashStore(), clk, ttl=ttl), clk


def test_uncontended_and_expiry_and_refresh():
    ls, clk = lease(ttl=1.0)
    assert ls.cas_put_if_absent_or_expired("job", "w0:5000") == (WON, 1, "w0:5000")
    assert ls.cas_put_if_absent_or_expired("job", "w1:5001")[:1] == (LOST,)
    assert ls.cas_put_if_absent_or_expired("job", "w1:5001")[2] == "w0:5000"
    clk.advance(0.5)
    assert ls.refresh("job", "w0:5000") == OK  # deadline extended to t + 1
    clk.advance(0.9)
    assert ls.cas_put_if_absent_or_expired("job", "w3:5003")[0] == LOST  # still valid
    clk.advance(0.2)  # past the refreshed deadline: expired
    assert ls.get("job") is None
    assert ls.cas_put_if_absent_or_expired("job", "w3:5003") == (WON, 2, "w3:5003")
    # the old leader's refresh after the re-election: NotLeader (address mismatch)
    assert ls.refresh("job", "w0:5000") == NOT
    assert ls.get("job")[0] == "w3:5003" and ls.get("job")[2] == 2


def test_erase_and_handoff():
    ls, clk = lease()
    ls.cas_put_if_absent_or_expired("job", "w0")
    assert ls.erase("job", "w1") == NOT  # non-leader: record unchanged
    assert ls.get("job")[0] == "w0"
    assert ls.erase("job", "w0") == OK  # graceful exit
    assert ls.get("job") is None
    assert ls.refresh("job", "w0") == NOT  # refresh of an erased record
    # next election proceeds immediately; generations keep increasing across the erase
    assert ls.cas_put_if_absent_or_expired("job", "w1") == (WON, 2, "w1")


def test_100_concurrent_candidates_exactly_one_wins():
    ls, _ = lease()
    out = [None] * 100
    go = threading.Barrier(100)

    def cand(i):
        go.wait()
        out[i] = ls.cas_put_if_absent_or_expired("job", f"w{i}")

    th = [threading.Thread(target=cand, args=(i,)) for i in range(100)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    won = [o for o in out if o[0] == WON]
    assert len(won) == 1 and won[0][1] == 1
    assert all(o[2] == won[0][2] for o in out)  # every loser sees the winner's address


def test_watch_delivers_elected_and_expired():
    ls, clk = lease(ttl=1.0)
    evs = []
    ls.watch("job", evs.append)
    ls.poll()
    assert evs == []  # no activity, no events
    ls.cas_put_if_absent_or_expired("job", "w0")
    assert evs == [("Elected", "job", "w0", 1)]
    clk.advance(1.05)  # leader killed: no refresh
    ls.poll()  # the ttl/10 expiry poll
    assert evs[-1] == ("Expired", "job", "", 0)
    ls.cas_put_if_absent_or_expired("job", "w2")
    assert evs[-1] == ("Elected", "job", "w2", 2)
    ls.erase("job", "w2")
    assert evs[-1] == ("Expired", "job", "", 0)


def test_random_interleavings_uniqueness_and_monotonic_generations():
    for seed in range(20):
        rng = random.Random(seed)
        ls, clk = lease(ttl=1.0)
        evs = []
        ls.watch("job", evs.append)
        holders = {}  # address -> generation it won
        for _ in range(300):
            a = f"w{rng.randrange(5)}"
            op = rng.random()
            if op < 0.4:
                st, gen, addr = ls.cas_put_if_absent_or_expired("job", a)
                if st == WON:
                    holders = {a: gen}
            elif op < 0.6:
                if ls.refresh("job", a) == OK:
                    assert a in holders
            elif op < 0.7:
                if ls.erase("job", a) == OK:
                    holders = {}
            else:
                clk.advance(rng.random() * 0.6)
                ls.poll()
            rec = ls.get("job")
            valid = [rec[0]] if rec else []
            assert len(valid) <= 1  # uniqueness
            if rec:
                assert rec[0] in holders
        gens = [e[3] for e in evs if e[0] == "Elected"]
        assert gens == sorted(gens) and len(set(gens)) == len(gens)  # strictly increasing


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _proc(rank, world, port, q):
    import time
    store = dist.TCPStore("127.0.0.1", port, world, rank == 0)
    ls = LeaderLease(store, ttl=30.0)
    st = dist.PrefixStore("sync/", store)
    r1 = ls.cas_put_if_absent_or_expired("job", f"w{rank}")
    st.set(f"r1/{rank}", r1[0])
    st.wait([f"r1/{r}" for r in range(world)])
    r2 = None
    if r1[0] == WON:  # the first leader leaves gracefully; the others elect a successor
        assert ls.erase("job", f"w{rank}") == OK
        st.set("erased", "1")
    else:
        st.wait(["erased"])
        r2 = ls.cas_put_if_absent_or_expired("job", f"w{rank}")
    q.put((rank, r1, r2))
    st.add("fin", 1)
    while rank == 0 and st.add("fin", 0) < world:  # the store server outlives the clients
        time.sleep(0.01)


def test_four_process_election_over_tcpstore():
    world, port = 4, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_proc, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    first = [r for r in res if r[1][0] == WON]
    assert len(first) == 1 and first[0][1][1] == 1
    second = [r for r in res if r[2] is not None and r[2][0] == WON]
    assert len(second) == 1 and second[0][2][1] == 2  # handoff: generation + 1
    assert second[0][0] != first[0][0]
