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
