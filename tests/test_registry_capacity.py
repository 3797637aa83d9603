"""Registries beyond the parameter-space recipe table (GPU).

The reference's DynamicsRegistry takes any number of (chain, params)
instances (proj/src/accelerated_lattice.cpp:10-41): e.g. per-region
Smagorinsky constants or wall velocities. The device keeps the first 16
recipes in kernel parameter space; larger registries (up to 256, the range of
the u8 slot array) run the KM_XREC kernels, which read the table from global
memory. Bit-identical to the oracle for every layout and decomposition.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from paper_2506_09242_b200 import _capi
from pyoracle import BB, BGK, COLLIDE, MBB, NODYN, RR, TRT, Recipe

pytestmark = pytest.mark.gpu


def many_recipes(n, rng):
    out = []
    for k in range(n):
        kind = k % 7
        if kind == 0:
            out.append(Recipe(kind=BB))
            continue
        if kind == 1:
            out.append(Recipe(kind=MBB, wall_velocity=(0.01 * (k % 5), -0.003 * (k % 3), 0.002)))
            continue
        if kind == 2 and k > 20:
            out.append(Recipe(kind=NODYN))
            continue
        base = (BGK, TRT, RR)[k % 3]
        r = Recipe(kind=COLLIDE, base=base, omega=1.0 + 0.9 * rng.random())
        if base == TRT:
            r.lambda_ = 0.1 + 0.2 * rng.random()
        if base == RR:
            r.omega_bulk_ho = 0.8 + 0.4 * rng.random()
        if k % 4 == 3 and base != RR:
            r.has_les, r.smagorinsky_c = True, 0.1 + 0.1 * rng.random()
        out.append(r)
    # keep every (chain, params) distinct so registration order == slot order
    seen = set()
    uniq = []
    for r in out:
        key = (r.chain_string(), tuple(r.params()))
        if key not in seen:
            seen.add(key)
            uniq.append(r)
    return uniq


def register(recipes):
    reg = dlb.DynamicsRegistry()
    for k, r in enumerate(recipes):
        p = np.asarray(r.params(), np.float64)
        slot = C.c_int32()
        _capi.check(_capi.lib().dlb_registry_register(reg.handle, r.chain_string().encode(),
                                                      p.ctypes.data if p.size else None, p.size, C.byref(slot)))
        assert slot.value == k
    return reg


@pytest.mark.parametrize("layout,slabs,precision", [("twopop", 1, 64), ("aa", 1, 64), ("twopop", 3, 64),
                                                    ("twopop", 1, 32)])
def test_large_registry_matches_oracle(oracle, layout, slabs, precision):
    rng = np.random.default_rng(7)
    recipes = many_recipes(170, rng)
    assert len(recipes) > 100
    dims, periodic = (18, 14, 12), (1, 1, 1)
    slot = rng.integers(0, len(recipes), size=(dims[2], dims[1], dims[0])).astype(np.int32)
    reg = register(recipes)
    dt = np.float64 if precision == 64 else np.float32
    n = int(np.prod(dims))
    rho = 1.0 + 0.01 * rng.standard_normal(n)
    u = [0.02 * rng.standard_normal(n) for _ in range(3)]
    f = oracle.fill_equilibrium(19, rho, *u, dt)
    want = oracle.step(19, dims, periodic, recipes, slot, f.copy(), 7)
    run = dlb.DeviceRun(dims, periodic, reg, q=19, precision=precision, slabs=slabs, layout=layout)
    run.fill_slots(slot)
    run.fill_state(rho, *u)
    run.exchange()
    assert "KM_XREC" in run.kernel_name()
    run.advance(7)
    assert np.array_equal(run.gather_populations(), want.astype(np.float64))


def test_large_registry_masked_sweep(oracle):
    """Masked sweep with > 16 instances: a solid box (bounce-back shell,
    NoDynamics core) inside randomly assigned collision / wall instances."""
    rng = np.random.default_rng(11)
    recipes = many_recipes(60, rng)
    nd = next(k for k, r in enumerate(recipes) if r.kind == NODYN)
    bb = next(k for k, r in enumerate(recipes) if r.kind == BB)
    live = [k for k, r in enumerate(recipes) if r.kind != NODYN]
    dims, periodic = (40, 12, 10), (1, 1, 1)
    slot = rng.choice(live, size=(dims[2], dims[1], dims[0])).astype(np.int32)
    slot[1:9, 1:11, 3:37] = bb
    slot[2:8, 2:10, 4:36] = nd
    reg = register(recipes)
    n = int(np.prod(dims))
    f = oracle.fill_equilibrium(19, np.ones(n), *[np.zeros(n)] * 3, np.float64)
    want = oracle.step(19, dims, periodic, recipes, slot, f.copy(), 5).reshape(19, -1)
    run = dlb.DeviceRun(dims, periodic, reg, q=19, precision=64, skip_nodynamics=True)
    run.fill_slots(slot)
    run.fill_state()
    run.advance(5)
    got = run.gather_populations().reshape(19, -1)
    active = np.asarray([recipes[s].kind != NODYN for s in slot.reshape(-1)])
    assert np.array_equal(got[:, active], want[:, active])
    # a NoDynamics cell next to a collision cell breaks the masked sweep's precondition
    slot[5, 5, 20] = live[3] if recipes[live[3]].kind == COLLIDE else live[2]
    slot[5, 5, 21] = nd
    slot[5, 5, 22] = next(k for k in live if recipes[k].kind == COLLIDE)
    with pytest.raises(dlb.ConfigError):
        run.fill_slots(slot)


def test_registry_beyond_slot_range_is_rejected():
    rng = np.random.default_rng(3)
    recipes = [Recipe(kind=COLLIDE, base=BGK, omega=1.0 + 0.9 * k / 300.0) for k in range(257)]
    reg = register(recipes)
    with pytest.raises(dlb.ConfigError) as e:
        dlb.DeviceRun((8, 8, 8), (1, 1, 1), reg)
    assert "256" in str(e.value)
