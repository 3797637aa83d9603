"""Ragged extents (nothing a multiple of a warp, a block or a TMA box): every
kernel family on odd, non-cubic lattices with mixed periodicity and a random
mix of fluid / wall / moving-wall / NoDynamics cells, against the CPU oracle
stepping the same initial state. Exact mode must be bit-identical on every
Collide-kind cell (and on all cells for the dense families)."""
import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from paper_2506_09242_b200.dolb import (CollisionParams, DeviceRun, DynamicsRegistry, LinkType,
                                        make_bounce_back, make_collision_chain, make_moving_bounce_back,
                                        make_no_dynamics)
from pyoracle import BGK, TRT, Oracle, Recipe, descriptor

pytestmark = pytest.mark.gpu
NODYN, BB, MBB, COLLIDE = 0, 1, 2, 3


def ragged_case(dims, periodic, seed, nodyn=False, base=TRT):
    """Registry + recipes in the same slot order, a random slot field, and a
    smooth random equilibrium state."""
    nx, ny, nz = dims
    rng = np.random.default_rng(seed)
    om, lam, uw = 1.63, 3.0 / 16.0, (0.03, -0.01, 0.02)
    lt = LinkType.TRT if base == TRT else LinkType.BGK
    reg = DynamicsRegistry()
    p = CollisionParams().set_trt(om, lam)
    chains = [make_collision_chain(lt, p), make_bounce_back(), make_moving_bounce_back(uw)]
    recipes = [Recipe(kind=COLLIDE, base=base, omega=om, lambda_=lam), Recipe(kind=BB),
               Recipe(kind=MBB, wall_velocity=uw)]
    if nodyn:
        chains.append(make_no_dynamics())
        recipes.append(Recipe(kind=NODYN))
    slots = [reg.register_chain(c) for c in chains]
    assert slots == list(range(len(chains)))
    slot = np.zeros((nz, ny, nx), np.int32)
    r = rng.random((nz, ny, nx))
    slot[r < 0.12] = 1
    slot[(r >= 0.12) & (r < 0.16)] = 2
    if nodyn:
        # a solid column plus random solid voxels; as in init_porous (cases.cpp:239-249)
        # a solid cell with any fluid neighbour bounces back, the others are NoDynamics
        zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        solid = ((xx - nx / 2) ** 2 / (nx / 3) ** 2 + (yy - ny / 2) ** 2 / (ny / 3) ** 2) < 1.0
        solid |= rng.random((nz, ny, nx)) < 0.25
        c = descriptor(19)[0]
        fluid_nb = np.zeros_like(solid)
        for i in range(1, 19):
            src = np.ones_like(solid)  # out-of-domain neighbours count as solid
            sl_dst = [slice(None)] * 3
            sl_src = [slice(None)] * 3
            shifted = solid
            for ax, cc in zip((2, 1, 0), (int(c[i][0]), int(c[i][1]), int(c[i][2]))):
                if cc == 0:
                    continue
                if periodic[2 - ax]:
                    shifted = np.roll(shifted, -cc, axis=ax)
                else:
                    tmp = np.ones_like(shifted)
                    if cc > 0:
                        tmp[(slice(None),) * ax + (slice(0, -1),)] = shifted[(slice(None),) * ax + (slice(1, None),)]
                    else:
                        tmp[(slice(None),) * ax + (slice(1, None),)] = shifted[(slice(None),) * ax + (slice(0, -1),)]
                    shifted = tmp
            fluid_nb |= ~shifted
        slot[:] = 0
        slot[solid & fluid_nb] = 1
        slot[solid & ~fluid_nb] = 3
    k = 2 * np.pi * rng.random(3)
    zz, yy, xx = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    rho = 1.0 + 0.01 * np.sin(xx * 0.3 + k[0]) * np.cos(yy * 0.2 + k[1])
    ux = 0.03 * np.sin(yy * 0.25 + k[1])
    uy = 0.02 * np.cos(zz * 0.3 + k[2])
    uz = 0.01 * np.sin(xx * 0.2 + k[0])
    return reg, recipes, slot, (rho.ravel(), ux.ravel(), uy.ravel(), uz.ravel())


def compare(run, recipes, slot, dims, periodic, steps, bits, fluid_only=False):
    f0 = run.gather_populations().copy()
    run.advance(steps)
    got = run.gather_populations().reshape(19, -1)
    f = f0.astype(np.float64 if bits == 64 else np.float32)
    Oracle().step(19, dims, periodic, recipes, slot, f, steps)
    want = np.asarray(f, np.float64).reshape(19, -1)
    sel = (slot.reshape(-1) == 0) if fluid_only else slice(None)
    d = np.abs(got[:, sel] - want[:, sel]).max()
    assert d == 0.0, d


DIMS = [((37, 19, 23), (1, 0, 1)), ((33, 45, 17), (0, 1, 1)), ((65, 7, 30), (1, 1, 0))]


@pytest.mark.parametrize("dims,periodic", DIMS)
@pytest.mark.parametrize("bits", [32, 64])
def test_ragged_dense(dims, periodic, bits):
    reg, recipes, slot, state = ragged_case(dims, periodic, 7)
    run = DeviceRun(dims, periodic, reg, precision=bits)
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, 9, bits)


@pytest.mark.parametrize("dims,periodic", DIMS)
def test_ragged_aa(dims, periodic):
    reg, recipes, slot, state = ragged_case(dims, periodic, 8)
    run = DeviceRun(dims, periodic, reg, precision=64, layout="aa")
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, 7, 64)


@pytest.mark.parametrize("dims,periodic", DIMS)
def test_ragged_zslabs(dims, periodic):
    reg, recipes, slot, state = ragged_case(dims, periodic, 9)
    run = DeviceRun(dims, periodic, reg, precision=32, slabs=3)
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, 8, 32)


@pytest.mark.parametrize("dims,periodic", DIMS)
def test_ragged_tma(dims, periodic):
    reg, recipes, slot, state = ragged_case(dims, periodic, 10)
    run = DeviceRun(dims, periodic, reg, precision=32, tma=True)
    run.fill(slot, state)
    assert "k_tma" in run.kernel_name()
    compare(run, recipes, slot, dims, periodic, 8, 32)


@pytest.mark.parametrize("dims,periodic", DIMS)
@pytest.mark.parametrize("variant", ["masked", "lists", "ballot"])
def test_ragged_porous_variants(dims, periodic, variant, monkeypatch):
    if variant == "ballot":
        monkeypatch.setenv("DLB_MASKED_COMPACT", "0")
    reg, recipes, slot, state = ragged_case(dims, periodic, 11, nodyn=True)
    run = DeviceRun(dims, periodic, reg, precision=64, skip_nodynamics=variant != "lists",
                    sparse_lists=variant == "lists")
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, 9, 64, fluid_only=True)


TINY = [((1, 1, 1), (1, 1, 1)), ((1, 2, 3), (1, 1, 1)), ((3, 1, 2), (1, 0, 1)), ((2, 3, 1), (0, 1, 1)),
        ((5, 4, 6), (0, 0, 0))]


@pytest.mark.parametrize("dims,periodic", TINY)
def test_tiny_lattices(dims, periodic):
    """Degenerate extents: single-cell periodic boxes (every link wraps onto the
    cell itself), one-plane axes, fully bounded boxes."""
    reg, recipes, slot, state = ragged_case(dims, periodic, 12)
    run = DeviceRun(dims, periodic, reg, precision=64)
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, 6, 64)


@pytest.mark.parametrize("slabs", [2, 4])
def test_one_plane_slabs(slabs):
    """z-slabs of a single plane (boundary launch only, no interior launch)."""
    dims, periodic = (6, 5, 4), (1, 1, 1)
    reg, recipes, slot, state = ragged_case(dims, periodic, 13)
    run = DeviceRun(dims, periodic, reg, precision=64, slabs=slabs)
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, 7, 64)


@pytest.mark.parametrize("steps", [2, 7, 10])
@pytest.mark.parametrize("dims,periodic", DIMS[:2] + TINY[:2])
def test_cooperative_multistep(dims, periodic, steps, monkeypatch):
    """Persistent cooperative sweep (k_pull_coop, opt-in DLB_COOP_MAX_CELLS):
    all steps of a call in one launch with grid-wide barriers, odd and even
    step counts (the state ends in either buffer)."""
    monkeypatch.setenv("DLB_COOP_MAX_CELLS", str(1 << 22))
    reg, recipes, slot, state = ragged_case(dims, periodic, 14)
    run = DeviceRun(dims, periodic, reg, precision=64)
    run.fill(slot, state)
    compare(run, recipes, slot, dims, periodic, steps, 64)
    run.advance(3)  # and again from the other buffer
    f = run.gather_populations()
    assert np.isfinite(f).all()


@pytest.mark.parametrize("bits,pinned", [(32, True), (32, False), (64, True)])
def test_ragged_host_block(bits, pinned):
    """The host-block drop-in (dlb_collide_and_stream on an AcceleratedBlock)
    on a ragged, partly periodic lattice with walls and a moving wall, through
    page-locked (pipelined) and pageable (staged) memory."""
    import ctypes as C
    from paper_2506_09242_b200 import _capi
    dims, periodic = (37, 19, 23), (1, 0, 1)
    nx, ny, nz = dims
    reg, recipes, slot, state = ragged_case(dims, periodic, 15)
    run = DeviceRun(dims, periodic, reg, precision=bits)
    run.fill(slot, state)
    f0 = run.gather_populations()
    dt = np.float32 if bits == 32 else np.float64
    want = f0.astype(dt).copy()
    Oracle().step(19, dims, periodic, recipes, slot, want, 3)
    shape = (19, nz + 2, ny + 2, nx + 2)
    nbytes = int(np.prod(shape)) * np.dtype(dt).itemsize
    p = C.c_void_p()
    if pinned:
        _capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
        blk = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(dt).reshape(shape)
        blk[:] = 0
    else:
        blk = np.zeros(shape, dt)
    try:
        blk[:, 1:-1, 1:-1, 1:-1] = f0.astype(dt).reshape(19, nz, ny, nx)
        tag = np.full(shape[1:], -1, np.int32)
        tag[1:-1, 1:-1, 1:-1] = np.vectorize(reg.tag_of_slot)(slot)
        pidx = np.full(shape[1:], -1, np.int32)
        pidx[1:-1, 1:-1, 1:-1] = slot
        for _ in range(3):
            dlb.refresh_envelope_periodic(blk, periodic)
            dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet.all_of(reg))
        got = blk[:, 1:-1, 1:-1, 1:-1].reshape(-1).astype(np.float64)
        assert np.array_equal(got, np.asarray(want, np.float64).reshape(-1))
    finally:
        if pinned:
            del blk
            _capi.lib().dlb_host_free(p)


def test_host_block_d3q27():
    """The host-block drop-in on a D3Q27 RR block (config 2's lattice)."""
    from paper_2506_09242_b200.dolb import make_collision_chain as mk
    from pyoracle import RR
    dims, periodic = (13, 11, 9), (1, 1, 1)
    nx, ny, nz = dims
    reg = DynamicsRegistry()
    p = CollisionParams().set_trt(1.71, 3.0 / 16.0)
    s0 = reg.register_chain(mk(LinkType.RR, p))
    recipes = [Recipe(kind=COLLIDE, base=RR, omega=1.71)]
    slot = np.zeros((nz, ny, nx), np.int32)
    rng = np.random.default_rng(3)
    state = (1.0 + 0.01 * rng.random(nx * ny * nz), 0.02 * rng.random(nx * ny * nz),
             0.01 * rng.random(nx * ny * nz), -0.01 * rng.random(nx * ny * nz))
    run = DeviceRun(dims, periodic, reg, q=27, precision=64)
    run.fill(slot + s0, state)
    f0 = run.gather_populations()
    want = f0.copy()
    Oracle().step(27, dims, periodic, recipes, slot, want, 2)
    shape = (27, nz + 2, ny + 2, nx + 2)
    blk = np.zeros(shape)
    blk[:, 1:-1, 1:-1, 1:-1] = f0.reshape(27, nz, ny, nx)
    tag = np.full(shape[1:], -1, np.int32)
    tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(s0)
    pidx = np.where(tag >= 0, s0, -1).astype(np.int32)
    for _ in range(2):
        dlb.refresh_envelope_periodic(blk, periodic, q=27)
        dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet.all_of(reg), q=27)
    assert np.array_equal(blk[:, 1:-1, 1:-1, 1:-1].reshape(-1), want.reshape(-1))
