"""One process per slab (here several processes sharing one B200): slabs
linked through CUDA IPC peer memory, halo pushed by the boundary-plane kernel,
progress flags in peer memory. The stitched result must equal the reference."""
import os
import subprocess
import sys

import numpy as np
import pytest

from pyoracle import canonical_hash

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,coll,L,steps,world", [("tgv16_bgk_f64", "BGK", 16, 10, 2),
                                                     ("cavity32_trt_f32", "TRT", 32, 200, 3)])
def test_ipc_slabs_bit_identical(golden, tmp_path, name, coll, L, steps, world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533",
           os.path.join(ROOT, "tests", "dist_gpu_worker.py"), str(tmp_path), str(L), str(steps), coll]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [np.load(tmp_path / f"rank{k}.npy").reshape(19, -1) for k in range(world)]
    full = np.concatenate(parts, axis=1).reshape(-1)
    assert canonical_hash(full) == golden[name]["sha256"]


def test_bench_two_ranks_protocol(tmp_path):
    """bench.py under torchrun at N=2 (both ranks on GPU 0, DLB_SAME_DEVICE):
    the driver's multi-GPU launch path prints one JSON line with the whole-job
    value, max-over-ranks timing and weak/strong scaling tag."""
    import json
    env = dict(os.environ, DLB_SAME_DEVICE="1")
    for cfg, L, scaling in (("c5", "128", "strong"), ("c3", "96", "weak")):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "bench.py"), "--gpus", "2",
               "--config", cfg, "--L", L, "--steps", "4", "--warmup", "3", "--no-cpu", "--no-e2e"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, r.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == scaling
        assert d["config"]["parallelism"] == "z-slab x2" and d["gpu_launches"] > 0
