"""bench.py's JSON contract on CPU: the reference arm (the CPU port of the MLP step at the
bench's batch, run on the host cores, plus the compiled reference's linear job) prints one parseable line with the driver's keys, and unmeasured figures are
emitted as null rather than NaN (json.dumps would write the non-JSON token NaN)."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_finite_replaces_nan_and_inf():
    import bench
    line = {"a": float("nan"), "b": [1.0, float("inf")], "c": {"d": 2.5, "e": -math.inf}}
    out = json.loads(json.dumps(bench._finite(line), allow_nan=False))
    assert out == {"a": None, "b": [1.0, None], "c": {"d": 2.5, "e": None}}


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"] == "mlp4096x8_bf16_b512_sgd"
    assert d["config"]["per_gpu_batch"] == 512 and d["config"]["same_config"]
    # the reference's own compiled C++ on its linear job (kind "reference"), when built here
    rl = d["reference_linear"]
    assert "unavailable" in rl or (rl["kind"] == "reference" and rl["value"] > 0)


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference"],
                       cwd=ROOT, capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr
