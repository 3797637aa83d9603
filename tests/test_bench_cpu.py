"""bench.py launch contract checks that need no GPU."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_rejects_world_mismatch():
    """A launcher that started a different number of ranks than --gpus asks
    for is an error, not a silent single-GPU number."""
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", DLB_BENCH_SPAWNED="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--no-cpu", "--no-e2e"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode != 0 and "--gpus 2" in r.stderr


def test_bench_spawn_command_uses_loopback():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    assert 1024 <= m.free_port() < 65536


def test_reference_arm_line():
    """bench.py --impl reference: one JSON line with the contract's keys (the
    reference compiled from its sources, timed on the host cores); rank > 0
    of a torchrun launch prints nothing and exits 0."""
    import json
    import pytest
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--L", "24", "--steps", "2",
           "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    if "unavailable" in line:
        pytest.skip(line["unavailable"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["metric"] == "MLUPS" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    r1 = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT,
                        env=dict(os.environ, RANK="1", WORLD_SIZE="2"))
    assert r1.returncode == 0 and r1.stdout.strip() == ""
