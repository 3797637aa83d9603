"""Multi-process host logic of the z-slab decomposition on CPU (gloo,
world_size 2 and 3): neighbour plan, balanced partition per rank and the
IPC-blob exchange that links slabs across processes."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_09242_b200.dolb import exchange_blobs, halo_neighbours, partition


def test_neighbour_plan():
    assert halo_neighbours(0, 1, True) == (None, None)
    assert halo_neighbours(0, 2, True) == (1, 1)
    assert halo_neighbours(0, 4, False) == (None, 1)
    assert halo_neighbours(3, 4, False) == (2, None)
    assert halo_neighbours(3, 4, True) == (2, 0)
    for w in (2, 3, 5, 8):
        for r in range(w):
            lo, up = halo_neighbours(r, w, True)
            assert halo_neighbours(lo, w, True)[1] == r and halo_neighbours(up, w, True)[0] == r


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blob = bytes([rank]) * (17 + rank)
        blobs = exchange_blobs(blob)
        lo, up = halo_neighbours(rank, world, True)
        z0, nz = partition(100, world)[rank]
        out.put((rank, [len(b) for b in blobs], blobs[lo][0], blobs[up][0], z0, nz))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_blob_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = partition(100, world)
    for rank, lens, lo_first, up_first, z0, nz in res:
        assert lens == [17 + r for r in range(world)]
        lo, up = halo_neighbours(rank, world, True)
        assert (lo_first, up_first) == (lo, up)
        assert (z0, nz) == parts[rank]
    assert sum(r[5] for r in res) == 100
