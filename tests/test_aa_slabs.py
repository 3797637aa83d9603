"""AA in-place streaming on linked z-slabs (GPU).

The AA pattern (one population array, half the memory of the reference's
two-population ping-pong, accelerated_lattice.hpp:83-85) on a decomposed domain
(multiblock.cpp:376-419): even steps touch only the cell's own locations, odd
steps read and write across the slab faces -- into the neighbour's boundary
plane through peer memory, with the pulled values pushed into the own ghost
plane by the neighbour's previous even step (k_aa). The stitched state must
equal the reference bit for bit after any step count (odd counts leave the
state in the face-crossing odd layout), for every slab count, and under the
same exchange-fault semantics as the two-population slabs.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from golden_cases import CASES, make_case
from pyoracle import BGK, RR, TRT, canonical_hash
from test_gpu_parity import product_setup

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,slabs", [("tgv16_bgk_f64", 2), ("tgv16_bgk_f64", 3), ("cavity32_trt_f32", 4),
                                        ("plates16_trt_vel_f64", 2), ("tgv32_rr_f32", 5),
                                        ("sphere48_trt_f64_c4", 3), ("cavity64_bgk_f64_c1", 8)])
def test_aa_zslabs_bit_identical_to_reference(golden, name, slabs):
    setup, bits, steps = product_setup(CASES[name])
    run = dlb.build_run(setup, precision=bits, slabs=slabs, layout="aa")
    run.advance(steps)
    assert "k_aa" in run.kernel_name()
    assert run.links(0)["upper"] != "none"
    assert canonical_hash(run.gather_populations()) == golden[name]["sha256"]


@pytest.mark.parametrize("spec,slabs", [
    (dict(kind="tgv", L=12, Re=50.0, Ma=0.1, collision=TRT, bits=64), 3),
    (dict(kind="cavity", L=18, Re=100.0, Ma=0.1, collision=BGK, bits=64), 2),
    (dict(kind="cavity", L=18, Re=100.0, Ma=0.1, collision=BGK, bits=64), 18),  # one-plane slabs
    (dict(kind="porous", L=12, Ma=0.01, collision=TRT, bits=32, plate_layers=4, upstream=3,
          downstream=3, drive="pressure"), 4),
    (dict(kind="tgv", L=14, Re=400.0, Ma=0.2, collision=RR, q=27, bits=64), 3),
])
def test_aa_zslabs_odd_and_even_counts_vs_oracle(oracle, spec, slabs):
    """Downloads after odd counts read the odd layout, whose face-crossing
    values sit in each slab's own ghost planes."""
    setup, bits, _ = product_setup(dict(spec, steps=0))
    run = dlb.build_run(setup, precision=bits, slabs=slabs, layout="aa")
    case = make_case(dict(spec, steps=0))
    dt = np.float64 if bits == 64 else np.float32
    f = oracle.initial_state(case, dt)
    dims, per, rec, slot = case.setup()
    for chunk in (1, 6, 1, 2, 5):  # odd, odd, even, even, odd totals; chunk 6 replays the 2-step graph
        run.advance(chunk)
        oracle.step(case.q, dims, per, rec, slot, f, chunk)
        assert np.array_equal(run.gather_populations(), f.astype(np.float64))


def test_aa_zslabs_checksums_and_macroscopic_match_two_population():
    cfg = dlb.CaseConfig(kind="tgv", L=24, Re=100.0, Ma=0.1)
    a = dlb.build_run(dlb.init_tgv(cfg), precision=32)
    b = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=4, layout="aa")
    for n in (3, 4):  # odd layout, then even
        a.advance(n)
        b.advance(n)
        assert a.checksum() == b.checksum()
        for x, y in zip(a.gather_macroscopic(), b.gather_macroscopic()):
            assert np.array_equal(x, y)


def test_aa_zslabs_upload_mid_run(oracle):
    case = make_case(dict(kind="tgv", L=10, Re=20.0, Ma=0.1, collision=BGK, bits=64, steps=0))
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    oracle.step(19, dims, per, rec, slot, f, 3)
    setup, _, _ = product_setup(dict(kind="tgv", L=10, Re=20.0, Ma=0.1, collision=BGK, bits=64, steps=0))
    run = dlb.build_run(setup, precision=64, slabs=2, layout="aa")
    run.advance(5)
    run.upload_populations(f)  # re-primes the ghost slots (exchange)
    assert np.array_equal(run.gather_populations(), f)
    run.advance(7)
    oracle.step(19, dims, per, rec, slot, f, 7)
    assert np.array_equal(run.gather_populations(), f)


def test_aa_zslab_memory_is_half_of_two_population():
    cfg = dlb.CaseConfig(kind="tgv", L=32, Re=100.0, Ma=0.1)
    a = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=2)
    b = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=2, layout="aa")
    pa, pb = a.traffic(0)[1], b.traffic(0)[1]
    assert pb < 0.55 * pa, (pa, pb)


def test_aa_zslab_silent_neighbour_fails_without_writing():
    """The exchange-fault contract of tests/test_exchange_fault.py on AA slabs:
    the slab that ran ahead keeps its last completed step."""
    cfg = dlb.CaseConfig(kind="tgv", L=16, Re=100.0, Ma=0.1)
    setup = dlb.init_tgv(cfg)
    run = dlb.build_run(setup, precision=64, slabs=2, layout="aa")
    run.set_halo_timeout(0.2)
    nxy = 16 * 16
    z0, nz0 = run.parts[0]
    run.step_slab(0, 2)  # slab 1 never steps: slab 0's step 2 waits in vain
    with pytest.raises(dlb.ExchangeError):
        run.synchronize()

    def mono(n):
        m = dlb.build_run(setup, precision=64)
        m.advance(n)
        return m.gather_populations().reshape(19, -1)

    got = run.gather_populations().reshape(19, -1)
    one = mono(1)
    # slab 0 after its one completed (odd, face-crossing) step; its values that
    # crossed into slab 1 are there too, so compare slab 0's own cells only
    sl = slice(z0 * nxy, (z0 + nz0) * nxy)
    assert np.array_equal(got[:, sl], one[:, sl])
    # recovery: slab 1 catches up, exchange clears the error, both continue
    run.step_slab(1, 1)
    run.synchronize()
    run.exchange()
    run.advance(3)
    run.synchronize()
    assert np.array_equal(run.gather_populations().reshape(19, -1), mono(4))


def test_aa_cannot_link_to_two_population():
    from paper_2506_09242_b200 import _capi
    from paper_2506_09242_b200.dolb import _Lattice, check
    reg = dlb.DynamicsRegistry()
    reg.register_chain(dlb.make_collision_chain(dlb.LinkType.BGK, dlb.CollisionParams(omega=1.2)))
    lats = []
    for k, layout in enumerate((_capi.LAYOUT_AA, 0)):
        d = _capi.LatticeDesc()
        d.dims[0], d.dims[1], d.dims[2] = 8, 8, 4
        d.q, d.precision_bits, d.layout = 19, 64, layout
        d.z_origin, d.global_nz = 4 * k, 8
        lats.append(_Lattice(d, reg))
    with pytest.raises(dlb.ConfigError):
        check(_capi.lib().dlb_lattice_link_local(lats[0].handle, lats[1].handle))


@pytest.mark.parametrize("world", [2, 3])
def test_aa_ipc_slabs_bit_identical(golden, tmp_path, world):
    """One process per AA slab (sharing one GPU here), linked through CUDA IPC."""
    env = dict(os.environ, DLB_WORKER_LAYOUT="aa")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29537",
           os.path.join(ROOT, "tests", "dist_gpu_worker.py"), str(tmp_path), "32", "200", "TRT"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    parts = [np.load(tmp_path / f"rank{k}.npy").reshape(19, -1) for k in range(world)]
    full = np.concatenate(parts, axis=1).reshape(-1)
    assert canonical_hash(full) == golden["cavity32_trt_f32"]["sha256"]


@pytest.mark.parametrize("layout", ["twopop", "aa"])
def test_group_graph_replays_match_single_slab(layout, monkeypatch):
    """dlb_lattices_step replays one CUDA graph with two steps of every slab;
    chunks of odd and even length (graph of the other parity -> one eager
    step), interleaved reads and a refill (new graph versions) must leave the
    state equal to the single-slab run."""
    monkeypatch.setenv("DLB_GROUP_GRAPH", "1")
    cfg = dlb.CaseConfig(kind="cavity", L=24, Re=100.0, Ma=0.1)
    setup = dlb.init_cavity(cfg)
    one = dlb.build_run(setup, precision=64)
    many = dlb.build_run(setup, precision=64, slabs=6, layout=layout)
    for chunk in (5, 16, 1, 9, 8, 20, 3):
        one.advance(chunk)
        many.advance(chunk)
        assert np.array_equal(one.gather_populations(), many.gather_populations()), chunk
    f = one.gather_populations()
    many.upload_populations(f)  # state write: same graph (versions unchanged), refilled buffers
    one.advance(17)
    many.advance(17)
    assert np.array_equal(one.gather_populations(), many.gather_populations())
