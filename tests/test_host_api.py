"""CPU-side checks of the product: the C-ABI library loads and exports every
symbol include/dlb.h declares; the host-side chain / registry / case layer
behaves like the reference (proj/tests/test_accelerated.cpp:56-115,
proj/src/chain.cpp); device entry points fail loudly without a GPU."""
import os
import re

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from paper_2506_09242_b200 import _capi
from paper_2506_09242_b200.dolb import (ChainLink, CollisionParams, DynamicsChain, DynamicsRegistry,
                                        LinkType, chain_string, make_collision_chain,
                                        make_regularized_velocity)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "dlb.h")).read()
    declared = set(re.findall(r"DLB_API\s+[\w\s\*]+?\b(dlb_\w+)\s*\(", header))
    assert len(declared) >= 30
    lib = _capi.lib()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_capi.EXPORTED), declared ^ set(_capi.EXPORTED)
    assert b"sm_100a" in lib.dlb_version()


def test_library_is_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def om(o):
    return CollisionParams(omega=o)


def test_registry_idempotent_and_sorted_tags():  # test_accelerated.cpp:56-75
    reg = DynamicsRegistry()
    bgk = make_collision_chain(LinkType.BGK, om(1.1))
    s = reg.register_chain(bgk)
    assert reg.register_chain(bgk) == s
    reg.register_chain(make_collision_chain(LinkType.TRT, om(1.2)))
    reg.register_chain(make_collision_chain(LinkType.RR, om(1.3), 0.16))
    assert reg.num_tags() == 3
    assert reg.tag_for("COLL_BGK") == 0
    assert reg.tag_for("COLL_TRT") == 1
    assert reg.tag_for("LES_Smagorinsky|COLL_RR") == 2
    for t in range(3):
        assert reg.tag_for(reg.chain_for(t)) == t
    with pytest.raises(dlb.ConfigError):
        reg.tag_for("COLL_RR")


def test_composite_boundary_chain():  # test_accelerated.cpp:77-95
    reg = DynamicsRegistry()
    ch = make_regularized_velocity(0, 1, (0.01, 0, 0), LinkType.TRT, om(1.0))
    assert chain_string(ch) == "Boundary_RegularizedVelocity_0_1__TRT"
    slot = reg.register_chain(ch)
    assert reg.chain_for(reg.tag_of_slot(slot)) == "Boundary_RegularizedVelocity_0_1__TRT"
    assert reg.slot_params(slot) == [0.01, 0.0, 0.0, 1.0, 3.0 / 16.0]
    three = DynamicsChain([ChainLink(LinkType.RegularizedVelocity, 0, 1), ChainLink(LinkType.Smagorinsky),
                           ChainLink(LinkType.RR)])
    assert chain_string(three) == "Boundary_RegularizedVelocity_0_1|LES_Smagorinsky|COLL_RR"


def test_same_string_different_params_share_tag():  # test_accelerated.cpp:97-107
    reg = DynamicsRegistry()
    a = reg.register_chain(make_collision_chain(LinkType.RR, om(1.3), 0.10))
    b = reg.register_chain(make_collision_chain(LinkType.RR, om(1.3), 0.17))
    assert a != b and reg.tag_of_slot(a) == reg.tag_of_slot(b)
    assert reg.slot_params(a)[0] == 0.10 and reg.slot_params(b)[0] == 0.17


def test_rejects_unknown_ids_and_unstable_rates():  # test_accelerated.cpp:109-115
    reg = DynamicsRegistry()
    with pytest.raises(dlb.ConfigError):
        reg.register_chain(DynamicsChain([ChainLink(LinkType.BGK)], dlb.ChainParams(om(2.5))))
    with pytest.raises(dlb.ConfigError):
        dlb.dolb._capi.get_string(_capi.lib().dlb_chain_canonical, b"COLL_XY")
    # malformed chains (chain.cpp:121-151)
    for bad in (b"COLL_BGK|COLL_TRT", b"LES_Smagorinsky|BounceBack", b"LES_Smagorinsky",
                b"Boundary_RegularizedVelocity_3_1__BGK", b""):
        with pytest.raises(dlb.ConfigError):
            _capi.get_string(_capi.lib().dlb_chain_canonical, bad)


CHAINS = ["COLL_BGK", "COLL_TRT", "COLL_RR", "NoDynamics", "BounceBack", "MovingBounceBack",
          "LES_Smagorinsky|COLL_BGK", "LES_Smagorinsky|COLL_RR",
          "Boundary_RegularizedVelocity_0_1|COLL_TRT", "Boundary_RegularizedPressure_2_M1__RR",
          "Boundary_RegularizedVelocity_1_M1|LES_Smagorinsky|COLL_BGK"]


@pytest.mark.parametrize("s", CHAINS)
def test_chain_strings_match_reference(reference, s):
    mine = _capi.get_string(_capi.lib().dlb_chain_canonical, s.encode())
    assert mine == reference.chain_roundtrip(s)


def test_omega_minus_matches_reference(reference):
    for om_, lam in ((1.2, 3 / 16), (1.7, 0.25), (0.6, 1 / 12)):
        assert dlb.dolb.derive_omega_minus(om_, lam) == reference.derive_omega_minus(om_, lam)


def test_partition_balanced_split():  # multiblock.cpp:24-31
    assert dlb.partition(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert dlb.partition(1024, 8) == [(128 * k, 128) for k in range(8)]
    with pytest.raises(ValueError):
        dlb.partition(3, 4)


@pytest.mark.parametrize("case", [
    dict(kind="cavity", L=16, Re=100.0, Ma=0.1),
    dict(kind="cavity", L=20, Re=1000.0, Ma=0.1, collision="TRT"),
    dict(kind="porous", L=16, Ma=0.01, collision="TRT", plate_layers=6, upstream=4, downstream=4),
    dict(kind="porous", L=16, Ma=0.01, collision="RR", plate_layers=5, upstream=3, downstream=2,
         drive="pressure"),
])
def test_case_generators_match_reference(reference, case):
    from pyoracle import Case
    lt = {"BGK": LinkType.BGK, "TRT": LinkType.TRT, "RR": LinkType.RR}
    oc = {"BGK": 0, "TRT": 1, "RR": 2}
    col = case.pop("collision", "BGK")
    cfg = dlb.CaseConfig(collision=lt[col], **case)
    setup = dlb.init_cavity(cfg) if cfg.kind == "cavity" else dlb.init_porous(cfg)
    tags, models = reference.tags(Case(collision=oc[col], **case))
    assert sorted({c.chain_string() for c in setup.chains}) == models  # registry tag order
    assert set(dlb.setup_models(setup)) <= set(models)
    names = [c.chain_string() for c in setup.chains]
    mine = np.asarray([models.index(n) for n in names])[setup.chain_index]
    assert np.array_equal(mine, tags)
    assert setup.dims == reference.dims(Case(collision=oc[col], **case))


def test_sphere_pack_generator(tmp_path):
    vox, phi = dlb.sphere_pack((40, 32, 24), radius=4.0, porosity=0.25, seed=7)
    vox2, _ = dlb.sphere_pack((40, 32, 24), radius=4.0, porosity=0.25, seed=7)
    assert np.array_equal(vox, vox2) and vox.shape == (24, 32, 40)
    assert set(np.unique(vox).tolist()) <= {0, 255}
    assert 0.2 < phi <= 0.25 and abs(phi - (vox == 0).mean()) < 1e-12
    p = tmp_path / "m.raw"
    vox.tofile(p)
    solid = dlb.load_voxels(str(p), (40, 32, 24))
    assert np.array_equal(solid, vox == 255)


def test_sphere_pack_loads_in_reference(reference, tmp_path):
    from pyoracle import Case
    vox, _ = dlb.sphere_pack((20, 16, 12), radius=3.0, porosity=0.3, seed=3)
    p = tmp_path / "m.raw"
    vox.tofile(p)
    case = dict(kind="porous", L=16, Ma=0.01, tau=1.0, geometry=str(p), voxel_dims=(20, 16, 12),
                upstream=3, downstream=3)
    tags, models = reference.tags(Case(collision=1, **case))
    cfg = dlb.CaseConfig(collision=LinkType.TRT, **case)
    setup = dlb.init_porous(cfg)
    mine = np.asarray([models.index(c.chain_string()) for c in setup.chains])[setup.chain_index]
    assert np.array_equal(mine, tags)


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    """The product path has no CPU fallback: creating a device lattice without
    a GPU raises instead of silently computing on the host."""
    reg = DynamicsRegistry()
    reg.register_chain(make_collision_chain(LinkType.BGK, om(1.5)))
    with pytest.raises(dlb.DlbError) as e:
        dlb.DeviceRun((8, 8, 8), (1, 1, 1), reg)
    assert e.value.status == 6


def test_refresh_envelope_periodic_matches_wrap():
    """dlb_refresh_envelope_periodic == refresh_envelope_periodic (host-only),
    every combination of periodic axes, one-plane and ragged extents; envelope
    cells of non-periodic axes keep what they held."""
    import itertools
    rng = np.random.default_rng(3)
    for (dt, shape), per in itertools.product(((np.float64, (5, 6, 7)), (np.float32, (1, 4, 3)),
                                               (np.float32, (3, 1, 9))),
                                              itertools.product((0, 1), repeat=3)):
        blk = rng.standard_normal((19,) + tuple(k + 2 for k in shape)).astype(dt)
        want = blk.copy()
        dlb.refresh_envelope_periodic(blk, per)
        # axis sweeps x, y, z with later axes spanning earlier ones (accelerated_lattice.cpp:202-238)
        if per[0]:
            want[:, 1:-1, 1:-1, 0] = want[:, 1:-1, 1:-1, -2]
            want[:, 1:-1, 1:-1, -1] = want[:, 1:-1, 1:-1, 1]
        if per[1]:
            want[:, 1:-1, 0, :] = want[:, 1:-1, -2, :]
            want[:, 1:-1, -1, :] = want[:, 1:-1, 1, :]
        if per[2]:
            want[:, 0] = want[:, -2]
            want[:, -1] = want[:, 1]
        assert np.array_equal(blk, want), (dt, shape, per)


def test_capi_null_arguments_and_buffer_protocol():
    """C-ABI conventions of proj/tests/test_capi.cpp:26-33 and :78-96: null
    arguments -> INVALID_ARGUMENT with a readable last error; string getters
    report the required size when called with a NULL buffer and refuse short
    buffers."""
    import ctypes as C
    lib = _capi.lib()
    assert b"." in lib.dlb_version()
    assert lib.dlb_registry_register(None, b"COLL_BGK", None, 0, None) == 1
    assert b"null" in lib.dlb_last_error()
    assert lib.dlb_lattice_step(None, 1) == 1
    assert lib.dlb_collide_and_stream(None, None, None, 0, 1) == 1
    assert lib.dlb_lattice_request_kinetic(None, None) == 1
    assert lib.dlb_lattice_reduce(None, None, None, None) == 1
    assert lib.dlb_refresh_envelope_periodic(None, None) == 1
    n = C.c_size_t()
    assert lib.dlb_chain_canonical(b"Boundary_RegularizedPressure_2_M1|COLL_RR", None, 0, C.byref(n)) == 0
    assert n.value == len("Boundary_RegularizedPressure_2_M1__RR") + 1
    small = C.create_string_buffer(4)
    assert lib.dlb_chain_canonical(b"COLL_BGK", small, 4, C.byref(n)) == 2
    assert b"buffer" in lib.dlb_last_error()
    full = C.create_string_buffer(n.value)
    assert lib.dlb_chain_canonical(b"COLL_BGK", full, n.value, C.byref(n)) == 0
    assert full.value == b"COLL_BGK"
    # a registry miss is a configuration error that names the chain
    reg = DynamicsRegistry()
    t = C.c_int32()
    assert lib.dlb_registry_tag_for(reg.handle, b"COLL_TRT", C.byref(t)) == 2
    assert b"COLL_TRT" in lib.dlb_last_error()
    # parameter records are validated against the chain (chain.cpp:188-230)
    slot = C.c_int32()
    two = (C.c_double * 2)(1.2, 0.5)
    assert lib.dlb_registry_register(reg.handle, b"COLL_BGK", two, 2, C.byref(slot)) == 2
    assert b"too long" in lib.dlb_last_error()
    assert lib.dlb_registry_register(reg.handle, b"COLL_TRT", two, 1, C.byref(slot)) == 2
    assert b"too short" in lib.dlb_last_error()


def test_last_error_is_thread_local():
    import threading
    lib = _capi.lib()
    lib.dlb_chain_canonical(b"NOT_A_LINK", None, 0, None)
    seen = {}

    def worker():
        lib.dlb_chain_canonical(b"COLL_BGK", None, 0, None)
        seen["msg"] = lib.dlb_last_error()
    th = threading.Thread(target=worker)
    th.start()
    th.join()
    assert b"NOT_A_LINK" in lib.dlb_last_error()
    assert b"NOT_A_LINK" not in seen["msg"]
