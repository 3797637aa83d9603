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


def test_bench_spawns_ranks_without_launcher():
    """`bench.py --gpus 2` without torchrun (the driver's plain form) starts two
    ranks itself and reports n_gpus 2; c5 is strong scaling (fixed L), c3 weak
    (L grows with the cube root of N: perfmodel.cpp:76-85). Every rank reports
    its halo links and bytes."""
    import json
    env = dict(os.environ, DLB_SAME_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    for cfg, L, scaling, want_L in (("c5", "128", "strong", 128), ("c3", "96", "weak", 121)):
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", cfg, "--L", L,
               "--steps", "4", "--warmup", "3", "--no-cpu", "--e2e-L", "64"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, r.stdout
        d = json.loads(lines[0])
        assert d["n_gpus"] == 2 and d["scaling"] == scaling and d["config"]["L"] == want_L
        ranks = d["config"]["halo"]["per_rank"]
        assert [x["rank"] for x in ranks] == [0, 1]
        for x in ranks:
            assert x["halo_bytes_per_step"] > 0
            if cfg == "c5":  # periodic ring: both neighbours linked (same GPU in this test)
                assert x["lower"] == x["upper"] == "same_gpu"
        if cfg == "c5":
            assert d["e2e"]["value"] > 0 and d["e2e"]["finite"]



def test_bench_two_aa_ranks():
    """`bench.py --gpus 2 --layout aa`: one AA in-place slab per rank, linked
    over CUDA IPC (odd steps store across the faces)."""
    import json
    env = dict(os.environ, DLB_SAME_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c5", "--L", "128",
           "--layout", "aa", "--steps", "4", "--warmup", "3", "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 2 and d["config"]["layout"] == "AA in-place SoA" and "k_aa" in d["config"]["kernel"]
    assert all(x["lower"] == x["upper"] == "same_gpu" for x in d["config"]["halo"]["per_rank"])
