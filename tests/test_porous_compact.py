"""Compacted porous sweep (k_cmp, GPU).

The masked porous sweep (DLB_FLAG_SKIP_NODYNAMICS: all-NoDynamics segments of
the sphere pack are never touched) stores its listed segments
and the segments they pull from in row-major compact arrays; the dense layout
is refreshed from them before every read. Bar: the reference's values on every
non-NoDynamics cell (collision and bounce-back), and the same state, checksums
and macroscopic fields as the uncompacted masked sweep (k_seg) at every read,
through graph-replayed and single-step advances, uploads and ragged extents.
"""
import dataclasses

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from golden_cases import CASES, make_case
from test_gpu_parity import product_setup

pytestmark = pytest.mark.gpu


def pair(setup, bits, monkeypatch):
    monkeypatch.setenv("DLB_POROUS_COMPACT", "1")
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    monkeypatch.setenv("DLB_POROUS_COMPACT", "0")
    ref = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    monkeypatch.delenv("DLB_POROUS_COMPACT")
    assert "k_cmp" in run.kernel_name(), run.kernel_name()
    assert "k_cmp" not in ref.kernel_name()
    return run, ref


@pytest.mark.parametrize("bits", [64, 32])
def test_compact_sweep_interleaved_reads_vs_oracle(oracle, bits, monkeypatch):
    spec = dict(CASES["sphere48_trt_f64_c4"], bits=bits)
    setup, _, _ = product_setup(spec)
    case = make_case(spec)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64 if bits == 64 else np.float32)
    run, ref = pair(setup, bits, monkeypatch)
    active = np.asarray(setup.chain_index).reshape(-1) != 2
    for chunk in (1, 1, 5, 2, 7, 1, 12):  # single steps and graph replays
        run.advance(chunk)
        ref.advance(chunk)
        oracle.step(19, dims, per, rec, slot, f, chunk)
        got = run.gather_populations().reshape(19, -1)
        assert np.array_equal(got[:, active], np.asarray(f, np.float64).reshape(19, -1)[:, active]), chunk
        assert np.array_equal(got, ref.gather_populations().reshape(19, -1))
        assert run.checksum(active_only=True) == ref.checksum(active_only=True)
        assert all(np.array_equal(a, b) for a, b in zip(run.gather_macroscopic(), ref.gather_macroscopic()))


def test_compact_sweep_restarts_after_upload(oracle, monkeypatch):
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, _ = product_setup(spec)
    case = make_case(spec)
    dims, per, rec, slot = case.setup()
    run, _ = pair(setup, bits, monkeypatch)
    run.advance(9)
    f = oracle.initial_state(case, np.float64)
    oracle.step(19, dims, per, rec, slot, f, 3)
    run.upload_populations(f)
    run.advance(6)
    oracle.step(19, dims, per, rec, slot, f, 6)
    active = np.asarray(setup.chain_index).reshape(-1) != 2
    got = run.gather_populations().reshape(19, -1)
    assert np.array_equal(got[:, active], f.reshape(19, -1)[:, active])


def sphere_setup(nx, ny, nz, periodic, seed, q=19, coll=dlb.LinkType.TRT):
    """Sphere pack (R = 3) with the reference's porous tagging rule in a box of
    any extent and periodicity: solids next to a fluid cell bounce back, the
    rest is NoDynamics (cases.cpp:239-249); a fluid buffer at both x ends."""
    vox, _ = dlb.sphere_pack((nx - 8, ny, nz), radius=3.0, porosity=0.3, seed=seed)
    cfg = dlb.CaseConfig(kind="porous", L=nx - 8, Ma=0.05, collision=coll, q=q, tau=0.8, upstream=4,
                         downstream=4)
    s = dlb.init_porous(cfg, solid=(vox == 255))
    if q == 27:  # init_porous tags with the D3Q19 neighbourhood: re-tag walls with all 26
        idx = np.asarray(s.chain_index).copy()
        solid = (idx == 1) | (idx == 2)
        fluid_nb = np.zeros_like(solid)
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    sh = np.roll(~solid, shift=(dz, dy), axis=(0, 1))
                    nb = np.zeros_like(solid)
                    if dx == 0:
                        nb = sh
                    elif dx == 1:
                        nb[:, :, 1:] = sh[:, :, :-1]
                    else:
                        nb[:, :, :-1] = sh[:, :, 1:]
                    fluid_nb |= nb
        idx[solid & fluid_nb] = 1
        idx[solid & ~fluid_nb] = 2
        s = dataclasses.replace(s, chain_index=idx)
    return dataclasses.replace(s, periodic=tuple(periodic))


@pytest.mark.parametrize("group_bytes", [8, 32, 64])
@pytest.mark.parametrize("nx,ny,nz,periodic", [
    (37, 20, 18, (0, 1, 1)),   # ragged x (partial last segment), the porous case's periodicity
    (40, 19, 21, (0, 0, 1)),   # non-periodic y: envelope rows are frozen sources
    (41, 22, 17, (0, 0, 0)),   # closed box
])
def test_compact_sweep_ragged_extents_match_masked(nx, ny, nz, periodic, group_bytes, monkeypatch):
    monkeypatch.setenv("DLB_SKIP_GROUP_BYTES", str(group_bytes))
    setup = sphere_setup(nx, ny, nz, periodic, seed=nx * ny + nz)
    run, ref = pair(setup, 64, monkeypatch)
    for chunk in (3, 8):
        run.advance(chunk)
        ref.advance(chunk)
        assert np.array_equal(run.gather_populations(), ref.gather_populations())


def test_compact_sweep_d3q27_and_fp32(monkeypatch):
    for q, bits in ((27, 64), (19, 32)):
        setup = sphere_setup(36, 16, 16, (0, 1, 1), seed=7, q=q)
        run, ref = pair(setup, bits, monkeypatch)
        run.advance(11)
        ref.advance(11)
        assert np.array_equal(run.gather_populations(), ref.gather_populations())


def test_compact_sweep_reports_launches_and_memory(monkeypatch):
    setup = sphere_setup(44, 24, 24, (0, 1, 1), seed=3)
    run, ref = pair(setup, 64, monkeypatch)
    assert run.traffic(0)[2] == 2            # main sweep + regularized inlet / outlet cells
    assert run.traffic(0)[1] > ref.traffic(0)[1]  # compact arrays beside the dense layout
    assert run.step_bytes() == ref.step_bytes()   # same algorithmic bytes (listed cells)


@pytest.mark.parametrize("flags", [{}, {"skip_nodynamics": True}, {"sparse_lists": True}])
def test_slots_replaced_by_uniform_slot(flags, monkeypatch):
    """A lattice whose porous slot field (regularized planes, NoDynamics
    solids: fix-up lists, segment lists, compact arrays, sparse lists) is
    replaced by one uniform slot steps exactly like a lattice built uniform."""
    monkeypatch.setenv("DLB_POROUS_COMPACT", "1")
    setup = sphere_setup(36, 16, 16, (0, 1, 1), seed=11)
    reg = dlb.DynamicsRegistry()
    slots = np.asarray([reg.register_chain(c) for c in setup.chains], np.int32)[setup.chain_index]
    bulk = int(slots[0, 0, 2])  # upstream fluid buffer: the bulk chain
    run = dlb.DeviceRun(setup.dims, setup.periodic, reg, precision=64, **flags)
    run.fill_slots(slots)
    run.fill_state()
    run.advance(3)
    run.fill_slots(bulk)
    run.fill_state()
    run.advance(9)
    ref = dlb.DeviceRun(setup.dims, setup.periodic, reg, precision=64)
    ref.fill_slots(bulk)
    ref.fill_state()
    ref.advance(9)
    assert np.array_equal(run.gather_populations(), ref.gather_populations())


@pytest.mark.parametrize("pack", ["1", "0"])
@pytest.mark.parametrize("block", ["32", "64", "128", "256"])
def test_segment_sweep_launch_variants(oracle, pack, block, monkeypatch):
    """The segment sweep's packed / linear entries and every block size give
    the reference's values on every non-NoDynamics cell, masked and dense."""
    monkeypatch.setenv("DLB_SEG_PACK", pack)
    monkeypatch.setenv("DLB_SEG_BLOCK", block)
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, steps = product_setup(spec)
    want = oracle.run_case(make_case(spec), np.float64, steps).reshape(19, -1)
    active = np.asarray(setup.chain_index).reshape(-1) != 2
    for skip in (True, False):
        run = dlb.build_run(setup, precision=bits, skip_nodynamics=skip)
        assert "k_seg" in run.kernel_name(), run.kernel_name()
        run.advance(steps)
        got = run.gather_populations().reshape(19, -1)
        if skip:
            assert np.array_equal(got[:, active], want[:, active])
        else:
            assert np.array_equal(got, want)


def test_masked_sweep_fast_mode_within_1e12(oracle):
    """FMA ("fast") arithmetic in the fused masked sweep: every non-NoDynamics
    population within the fp64 bar (max raw-relative error 1e-12)."""
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True, arith="fast")
    assert "k_seg" in run.kernel_name() and "fast" in run.kernel_name()
    run.advance(steps)
    got = run.gather_populations().reshape(19, -1)
    want = oracle.run_case(make_case(spec), np.float64, steps).reshape(19, -1)
    active = np.asarray(setup.chain_index).reshape(-1) != 2
    w = np.asarray(__import__("pyoracle").descriptor(19)[1])[:, None]
    rel = np.abs(got[:, active] - want[:, active]) / (np.abs(want[:, active]) + w)
    assert rel.max() <= 1e-12
