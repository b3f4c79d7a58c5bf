"""Multi-GPU (one process per GPU) parity of the fused NVLink allreduce + update path.
Runs tests/mp_parity_worker.py under torch.distributed.run on every visible GPU (>= 2)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


# overlap: "" = default (3 when the layers split into per-GPU row blocks, else 0), 0 = one
# fused collective kernel after the backward, 1 = per-layer collective kernels on a side
# stream, 2 = per-layer copy-engine transfers + shard updates, 3 = reduce-scatter in the
# wgrad GEMM epilogues + per-layer shard update / all-gather.  "3/defer" runs mode 3's push
# collective on a side stream overlapping the next forward (EDL_AG_DEFER=1, per-layer flags);
# "3/defer-ce" does the all-gather half on the copy engines under the next forward
# (EDL_AG_DEFER=2: local shard update after the backward, per-layer peer copies + flags).
# 4 = the whole exchange (reduce-scatter, sharded SGD, weight all-gather) inside the
# weight-gradient GEMMs, per-tile arrival counters across GPUs.
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
@pytest.mark.parametrize("overlap", ["", "0", "1", "2", "3", "3/defer", "3/defer-ce", "4", "5", "6"])
def test_two_or_more_gpus_match_oracle(overlap):
    n = min(torch.cuda.device_count(), 4)
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(here, "mp_parity_worker.py")]
    env = dict(os.environ)
    env.pop("EDL_OVERLAP", None)
    env.pop("EDL_AG_DEFER", None)
    if "/defer" in overlap:
        env["EDL_AG_DEFER"] = "2" if overlap.endswith("-ce") else "1"
        overlap = overlap.split("/")[0]
    if overlap:
        env["EDL_OVERLAP"] = overlap
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP-PARITY OK" in p.stdout


# Scale-in across processes: the upper half of the ring leaves at t=4 (every process
# schedules the event; the leavers' processes get Exit at the switch), checked against the
# oracle driving the same event (linear job bit-exact, MLP within the static tolerances).
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_multi_process_scale_in():
    n = min(torch.cuda.device_count(), 4)
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29537",
           os.path.join(here, "mp_scale_in_worker.py")]
    env = dict(os.environ)
    env.pop("EDL_OVERLAP", None)
    env.pop("EDL_AG_DEFER", None)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP-SCALE-IN OK" in p.stdout


# Stop-free scale-out across processes: the upper half of the ranks join at t=4 through
# Job.joining (built while the ring trains, model copied in over NVLink at the switch),
# checked against the oracle driving the same event.
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_multi_process_scale_out():
    n = min(torch.cuda.device_count(), 4)
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29539",
           os.path.join(here, "mp_scale_out_worker.py")]
    env = dict(os.environ)
    env.pop("EDL_OVERLAP", None)
    env.pop("EDL_AG_DEFER", None)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP-SCALE-OUT OK" in p.stdout


# Scheduler-facing scaling across processes (paper_1909_11985_b200/control.py): scale_out
# with Ready -> switch_t = t + max(k, margin) agreed through the rendezvous store, Retry while
# pending, momentum carried to the newcomers, straggler detection over the processes' published
# mini-batch times and the leader's scale_in, all checked against the oracle.
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_multi_process_scheduler_facing_scaling():
    n = min(torch.cuda.device_count(), 4)
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29541",
           os.path.join(here, "mp_elastic_api_worker.py")]
    env = dict(os.environ)
    env.pop("EDL_OVERLAP", None)
    env.pop("EDL_AG_DEFER", None)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=400, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP-ELASTIC-API OK" in p.stdout
    print([ln for ln in p.stdout.splitlines() if "MP-ELASTIC-API" in ln])


# Consistent failure recovery across processes: collective checkpoint at t=5, the last rank's
# process dies after t=8, the survivors drop its replica, reload the checkpoint and go on --
# least squares bit-exact with the oracle's snapshot / restore, MLP (momentum) within 1e-3.
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_multi_process_consistent_recovery():
    n = min(torch.cuda.device_count(), 4)
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29543",
           os.path.join(here, "mp_recovery_worker.py")]
    env = dict(os.environ)
    env.pop("EDL_OVERLAP", None)
    env.pop("EDL_AG_DEFER", None)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=400, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP-RECOVERY OK" in p.stdout


# Leader election and handoff across processes (control.LeaderLease over the rendezvous
# store): the elected leader scales itself in, the survivor wins the next election
# (generation 2) and scales the old leader's process back out -- checked against the oracle.
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs >= 2 GPUs")
def test_multi_process_leader_handoff():
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29545",
           os.path.join(here, "mp_leader_handoff_worker.py")]
    env = dict(os.environ)
    env.pop("EDL_OVERLAP", None)
    env.pop("EDL_AG_DEFER", None)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=400, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "MP-HANDOFF OK" in p.stdout
