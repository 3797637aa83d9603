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
