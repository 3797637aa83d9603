"""Exchange failure detection of linked z-slabs (GPU).

The reference makes a lost or duplicated halo frame fatal: ExchangeError from
exchange_recv before the step writes anything (proj/src/multiblock.cpp:305-345;
FaultyTransport, proj/tests/test_multiblock.cpp:23-51, 258-274). The device
analogue: a neighbour that never finishes its boundary planes makes the halo
wait time out; that step and every later queued one write nothing,
DLB_ERROR_EXCHANGE is reported, and the slab is left at its last completed
step. dlb_lattice_exchange clears the error once the slabs agree again.
"""
import numpy as np
import pytest

import paper_2506_09242_b200 as dlb

pytestmark = pytest.mark.gpu


def tgv(L=16):
    cfg = dlb.CaseConfig(kind="tgv", L=L, Re=100.0, Ma=0.1)
    return dlb.init_tgv(cfg)


def mono_after(setup, steps):
    run = dlb.build_run(setup, precision=64)
    run.advance(steps)
    return run.gather_populations().reshape(19, -1)


@pytest.mark.parametrize("steps", [3, 6])  # 6: the failing steps replay from the captured graph
def test_silent_neighbour_fails_without_writing(steps):
    setup = tgv(16)
    run = dlb.build_run(setup, precision=64, slabs=2)
    run.set_halo_timeout(0.2)
    nxy = 16 * 16
    z0, nz0 = run.parts[0]
    run.step_slab(0, steps)  # slab 1 never steps: slab 0's step 2 waits for it in vain
    with pytest.raises(dlb.ExchangeError) as e:
        run.synchronize()
    assert "timed out" in str(e.value)
    got = run.gather_populations().reshape(19, -1)
    one = mono_after(setup, 1)
    zero = mono_after(setup, 0)
    # slab 0 kept the state after its one completed step, slab 1 is untouched
    assert np.array_equal(got[:, z0 * nxy:(z0 + nz0) * nxy], one[:, z0 * nxy:(z0 + nz0) * nxy])
    assert np.array_equal(got[:, (z0 + nz0) * nxy:], zero[:, (z0 + nz0) * nxy:])


def test_recovery_after_exchange():
    setup = tgv(16)
    run = dlb.build_run(setup, precision=64, slabs=2)
    run.set_halo_timeout(0.2)
    run.step_slab(0, 2)
    with pytest.raises(dlb.ExchangeError):
        run.synchronize()
    run.step_slab(1, 1)  # the lagging slab catches up to step 1
    run.synchronize()
    run.exchange()  # clears the error, re-primes the ghosts of the common state
    run.advance(2)
    run.synchronize()
    assert np.array_equal(run.gather_populations().reshape(19, -1), mono_after(setup, 3))


def test_timeout_validation():
    run = dlb.build_run(tgv(16), precision=64, slabs=2)
    with pytest.raises(dlb.ConfigError):
        run.set_halo_timeout(0.0)
