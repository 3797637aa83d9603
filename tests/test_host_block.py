"""dlb_collide_and_stream on host AcceleratedBlock arrays (GPU): the
reference's two-array swap contract and the per-shape device cache.

Reference: collide_and_stream<T> writes f_out then swaps f_in / f_out
(proj/src/accelerated_lattice.cpp:157-200); the hybrid loop refreshes the
envelope of the new f_in before every step (proj/tests/test_accelerated.cpp:171-186).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from paper_2506_09242_b200 import _capi
from pyoracle import BGK, TRT, Case

pytestmark = pytest.mark.gpu


def pinned(shape, dtype):
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    p = C.c_void_p()
    _capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
    arr = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(dtype).reshape(shape)
    arr[:] = 0
    return arr, p


def tgv_block(n, reg, dtype, alloc):
    case = Case(kind="tgv", L=n, Re=50.0, Ma=0.1, collision=BGK)
    s = reg.register_chain(dlb.init_tgv(dlb.CaseConfig(kind="tgv", L=n, Re=50.0, Ma=0.1)).chains[0])
    blk, keep = alloc((19, n + 2, n + 2, n + 2), dtype)
    tag = np.full((n + 2,) * 3, -1, np.int32)
    tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(s)
    pidx = np.where(tag >= 0, s, -1).astype(np.int32)
    return case, blk, keep, tag, pidx


def host_alloc(shape, dtype):
    return np.zeros(shape, dtype), None


@pytest.mark.parametrize("memory", ["pageable", "pinned"])
def test_two_array_swap_contract(oracle, memory):
    n, steps = 12, 4
    alloc = pinned if memory == "pinned" else host_alloc
    reg = dlb.DynamicsRegistry()
    case, a, ka, tag, pidx = tgv_block(n, reg, np.float64, alloc)
    b, kb = alloc(a.shape, np.float64)
    dims, per, rec, slot = case.setup()
    f0 = oracle.initial_state(case, np.float64)
    a[:, 1:-1, 1:-1, 1:-1] = f0.reshape(19, n, n, n)
    try:
        f_in, f_out = a, b
        want = f0.copy()
        for _ in range(steps):
            prev = f_in[:, 1:-1, 1:-1, 1:-1].copy()
            dlb.refresh_envelope_periodic(f_in, (1, 1, 1))
            f_in, f_out = dlb.collide_and_stream(reg, f_in, tag, pidx, dlb.DispatchSet.all_of(reg), f_out=f_out)
            want = oracle.step(19, dims, per, rec, slot, want, 1)
            assert np.array_equal(f_in[:, 1:-1, 1:-1, 1:-1].reshape(-1), want)
            assert np.array_equal(f_out[:, 1:-1, 1:-1, 1:-1], prev)  # the previous state, untouched
        assert f_in is (a if steps % 2 == 0 else b)
        # a dispatch error leaves both arrays alone
        before = (f_in.copy(), f_out.copy())
        with pytest.raises(dlb.DispatchError):
            dlb.collide_and_stream(reg, f_in, tag, pidx, dlb.DispatchSet(), f_out=f_out)
        assert np.array_equal(f_in, before[0]) and np.array_equal(f_out, before[1])
    finally:
        for k in (ka, kb):
            if k is not None:
                _capi.lib().dlb_host_free(k)


def test_device_cache_follows_registry_content(oracle):
    """The per-shape device context is tied to the registry's content: a freed
    registry drops its entries, and a new registry (possibly at the same
    address, same instance count, other parameters) never reuses stale recipes."""
    n = 10
    dlb.block_cache_release()
    assert dlb.block_cache_info()[0] == 0
    for omega in (1.2, 1.7):
        reg = dlb.DynamicsRegistry()
        s = reg.register_chain(dlb.make_collision_chain(dlb.LinkType.TRT, dlb.CollisionParams().set_trt(omega, 3 / 16)))
        case = Case(kind="tgv", L=n, Re=50.0, Ma=0.1, collision=TRT)
        dims, per, _, slot = case.setup()
        rec = case.bulk_recipe()
        rec.omega = omega
        f0 = oracle.initial_state(case, np.float64)
        want = oracle.step(19, dims, per, [rec], slot, f0.copy(), 1)
        blk = np.zeros((19, n + 2, n + 2, n + 2))
        blk[:, 1:-1, 1:-1, 1:-1] = f0.reshape(19, n, n, n)
        tag = np.full((n + 2,) * 3, -1, np.int32)
        tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(s)
        pidx = np.where(tag >= 0, s, -1).astype(np.int32)
        dlb.refresh_envelope_periodic(blk, (1, 1, 1))
        dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet.all_of(reg))
        assert np.array_equal(blk[:, 1:-1, 1:-1, 1:-1].reshape(-1), want), omega
        entries, dev_bytes = dlb.block_cache_info()
        assert entries == 1 and dev_bytes > 0
        del reg  # dlb_registry_free drops the registry's cache entries
        assert dlb.block_cache_info()[0] == 0


def test_cache_release_frees_device_memory():
    reg = dlb.DynamicsRegistry()
    n = 16
    _, blk, _, tag, pidx = tgv_block(n, reg, np.float32, host_alloc)
    dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet.all_of(reg))
    assert dlb.block_cache_info()[0] == 1
    dlb.block_cache_release()
    assert dlb.block_cache_info() == (0, 0)
    dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet.all_of(reg))  # rebuilt on demand
    assert dlb.block_cache_info()[0] == 1


def _envelope_mask(shape):
    m = np.ones(shape, bool)
    m[:, 1:-1, 1:-1, 1:-1] = False
    return m


@pytest.mark.parametrize("memory", ["pageable", "pinned"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_envelope_after_step(memory, dtype):
    """step_range writes interior cells only (accelerated_lattice.cpp:126-153).
    In place, the caller's envelope survives the step on both paths. Into f_out:
    the pageable path leaves f_out's envelope untouched; the pinned pipeline
    copies whole planes back, whose x / y envelope cells carry f_in's envelope
    (never stale device memory), and the z envelope planes are not written."""
    n, sentinel = 12, 1234.5
    alloc = pinned if memory == "pinned" else host_alloc
    reg = dlb.DynamicsRegistry()
    case, a, ka, tag, pidx = tgv_block(n, reg, dtype, alloc)
    b, kb = alloc(a.shape, dtype)
    try:
        a[:, 1:-1, 1:-1, 1:-1] = 0.01  # a uniform (non-equilibrium) state: any finite values do
        dlb.refresh_envelope_periodic(a, (1, 1, 1))
        a[:, 1:-1, 0, :] = 0.5   # x / y envelope of the interior planes differs from f_out's
        env = _envelope_mask(a.shape)
        b[:] = sentinel
        before_a = a.copy()
        new, old = dlb.collide_and_stream(reg, a, tag, pidx, dlb.DispatchSet.all_of(reg), f_out=b)
        assert new is b and old is a
        assert np.array_equal(old, before_a)
        interior = new[:, 1:-1, 1:-1, 1:-1]
        assert np.all(np.isfinite(interior)) and not np.any(interior == sentinel)
        assert np.all(new[:, 0] == sentinel) and np.all(new[:, -1] == sentinel)  # z envelope planes
        xy = np.zeros(a.shape, bool)
        xy[:, 1:-1] = env[:, 1:-1]
        if memory == "pageable":
            assert np.all(new[env] == sentinel)
        else:
            assert np.array_equal(new[xy], before_a[xy])
        # in place: the envelope of f_in is left as the caller set it
        a[env] = -sentinel
        got = dlb.collide_and_stream(reg, a, tag, pidx, dlb.DispatchSet.all_of(reg))
        assert got is a and np.all(a[env] == -sentinel)
    finally:
        for k in (ka, kb):
            if k is not None:
                _capi.lib().dlb_host_free(k)


def test_pinned_ragged_block_matches_pageable():
    """A ragged block (x, y, z extents differ, x not a multiple of the warp)
    through the pinned pipeline equals the pageable path bit for bit: every
    state's interior, and the previous state (f_out) entirely."""
    nx, ny, nz = 37, 11, 9
    reg = dlb.DynamicsRegistry()
    s = reg.register_chain(dlb.init_tgv(dlb.CaseConfig(kind="tgv", L=8, Re=50.0, Ma=0.1)).chains[0])
    shape = (19, nz + 2, ny + 2, nx + 2)
    tag = np.full(shape[1:], -1, np.int32)
    tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(s)
    pidx = np.where(tag >= 0, s, -1).astype(np.int32)
    rng = np.random.default_rng(7)
    init = (rng.standard_normal(shape) * 1e-3).astype(np.float64)
    outs = []
    keep = []
    try:
        for alloc in (host_alloc, pinned):
            a, ka = alloc(shape, np.float64)
            b, kb = alloc(shape, np.float64)
            keep += [ka, kb]
            a[:] = init
            b[:] = 7.0
            f_in, f_out = a, b
            for _ in range(3):
                dlb.refresh_envelope_periodic(f_in, (1, 1, 1))
                f_in, f_out = dlb.collide_and_stream(reg, f_in, tag, pidx, dlb.DispatchSet.all_of(reg), f_out=f_out)
            outs.append((f_in.copy(), f_out.copy()))
        (pa_new, pa_old), (pi_new, pi_old) = outs
        assert np.array_equal(pa_new[:, 1:-1, 1:-1, 1:-1], pi_new[:, 1:-1, 1:-1, 1:-1])
        assert np.array_equal(pa_old, pi_old)
    finally:
        for k in keep:
            if k is not None:
                _capi.lib().dlb_host_free(k)


@pytest.mark.parametrize("plane", [1, 5, 12])
@pytest.mark.parametrize("in_place", [True, False])
def test_single_cell_slot_change_in_uniform_row(plane, in_place):
    """The scan summarises uniform rows of the cached slots by one value, and
    on a cached pinned block compares param_index plane by plane beside the
    copy-back (which it gates chunk by chunk). A one-cell slot change in the
    first / a middle / the last plane must recompute from that plane's chunk:
    the result equals a step from a freshly built device context, and the
    change matters."""
    n = 12
    reg = dlb.DynamicsRegistry()
    case, a, ka, tag, pidx = tgv_block(n, reg, np.float64, pinned)
    b, kb = pinned(a.shape, np.float64)
    s2 = reg.register_chain(dlb.init_tgv(dlb.CaseConfig(kind="tgv", L=n, Re=5.0, Ma=0.1)).chains[0])
    alld = dlb.DispatchSet.all_of(reg)

    def step(src, t, p):
        dlb.refresh_envelope_periodic(src, (1, 1, 1))
        if in_place:
            return dlb.collide_and_stream(reg, src, t, p, alld).copy()
        new, _ = dlb.collide_and_stream(reg, src, t, p, alld, f_out=b)
        return new.copy()

    try:
        a[:, 1:-1, 1:-1, 1:-1] = 0.01
        rng = np.random.default_rng(3)
        a[:, 1:-1, 1:-1, 1:-1] += rng.standard_normal((19, n, n, n)) * 1e-4
        for _ in range(2):
            dlb.refresh_envelope_periodic(a, (1, 1, 1))
            dlb.collide_and_stream(reg, a, tag, pidx, alld)
        snap = a.copy()
        tag2, pidx2 = tag.copy(), pidx.copy()
        tag2[plane, 7, 3], pidx2[plane, 7, 3] = reg.tag_of_slot(s2), s2
        cached = step(a, tag2, pidx2)                       # cached context, gated copy-back
        dlb.block_cache_release()
        a[:] = snap
        fresh = step(a, tag2, pidx2)                        # fresh context
        assert np.array_equal(cached[:, 1:-1, 1:-1, 1:-1], fresh[:, 1:-1, 1:-1, 1:-1])
        a[:] = snap
        same = step(a, tag, pidx)
        near = (slice(None), slice(plane - 1, plane + 2), slice(6, 9), slice(2, 5))
        assert not np.array_equal(cached[near], same[near])  # the changed cell matters
        far = (slice(None), slice(1, -1), slice(1, 4), slice(8, -1))
        assert np.array_equal(cached[far], same[far])
    finally:
        for k in (ka, kb):
            _capi.lib().dlb_host_free(k)


@pytest.mark.parametrize("memory", ["pageable", "pinned"])
def test_unregistered_slot_rejected_then_recovers(memory):
    """A param_index naming an unregistered slot is rejected (the reference
    would index past its recipe table); the cached context must not keep the
    rejected slots, so the next valid call steps with the right ones."""
    n = 12
    alloc = pinned if memory == "pinned" else host_alloc
    reg = dlb.DynamicsRegistry()
    case, a, ka, tag, pidx = tgv_block(n, reg, np.float64, alloc)
    s2 = reg.register_chain(dlb.init_tgv(dlb.CaseConfig(kind="tgv", L=n, Re=5.0, Ma=0.1)).chains[0])
    alld = dlb.DispatchSet.all_of(reg)
    try:
        a[:, 1:-1, 1:-1, 1:-1] = 0.01
        for _ in range(2):
            dlb.refresh_envelope_periodic(a, (1, 1, 1))
            dlb.collide_and_stream(reg, a, tag, pidx, alld)
        snap = a.copy()
        bad = pidx.copy()
        bad[9, 4, 4] = 99
        with pytest.raises(Exception):
            dlb.collide_and_stream(reg, a, tag, bad, alld)
        tag2, pidx2 = tag.copy(), pidx.copy()
        tag2[9, 4, 4], pidx2[9, 4, 4] = reg.tag_of_slot(s2), s2
        a[:] = snap
        dlb.refresh_envelope_periodic(a, (1, 1, 1))
        got = dlb.collide_and_stream(reg, a, tag2, pidx2, alld).copy()
        dlb.block_cache_release()
        a[:] = snap
        dlb.refresh_envelope_periodic(a, (1, 1, 1))
        want = dlb.collide_and_stream(reg, a, tag2, pidx2, alld)
        assert np.array_equal(got[:, 1:-1, 1:-1, 1:-1], want[:, 1:-1, 1:-1, 1:-1])
    finally:
        if ka is not None:
            _capi.lib().dlb_host_free(ka)


def test_pinned_pipeline_uses_the_lattice_buffers():
    """The pinned pipeline's host-layout mirrors live in the cached lattice's
    own two population buffers: a host-block context costs one two-population
    lattice (+ staging), not a second pair of state-sized buffers."""
    import torch
    n = 192
    reg = dlb.DynamicsRegistry()
    _, a, ka, tag, pidx = tgv_block(n, reg, np.float32, pinned)
    b, kb = pinned(a.shape, np.float32)
    try:
        dlb.block_cache_release()
        torch.cuda.init()
        torch.cuda.synchronize()
        free0 = torch.cuda.mem_get_info()[0]
        a[:, 1:-1, 1:-1, 1:-1] = 0.01
        dlb.refresh_envelope_periodic(a, (1, 1, 1))
        dlb.collide_and_stream(reg, a, tag, pidx, dlb.DispatchSet.all_of(reg), f_out=b)
        dlb.refresh_envelope_periodic(b, (1, 1, 1))
        dlb.collide_and_stream(reg, b, tag, pidx, dlb.DispatchSet.all_of(reg), f_out=a)  # cached: pinned pipeline
        used = free0 - torch.cuda.mem_get_info()[0]
        lattice_bytes = dlb.block_cache_info()[1]
        mirror_pair = 2 * a.nbytes
        assert used < lattice_bytes + mirror_pair // 2, (used, lattice_bytes, mirror_pair)
    finally:
        dlb.block_cache_release()
        for k in (ka, kb):
            _capi.lib().dlb_host_free(k)
