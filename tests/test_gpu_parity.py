"""GPU parity: the sm_100a collide-and-stream path (through the C ABI) against
the reference's outputs and the CPU oracle on the same inputs.

Bar (BASELINE.json north_star): exact-arithmetic mode is bit-identical
(max |diff| = 0) for fp64 and fp32 on D3Q19; the FMA ("fast") mode stays
within max raw-relative error 1e-12 per population in fp64 and, in fp32,
5e-5 per population with |d rho|, |d u| <= 1e-5.
D3Q27 has no reference: it is compared with the oracle's restatement.
"""
import os

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb
from golden_cases import CASES, SPHERE_RAW
from paper_2506_09242_b200.dolb import LinkType
from pyoracle import BGK, RR, TRT, Case, canonical_hash, descriptor

pytestmark = pytest.mark.gpu

LT = {0: LinkType.BGK, 1: LinkType.TRT, 2: LinkType.RR}


def product_setup(spec):
    s = dict(spec)
    bits, steps = s.pop("bits"), s.pop("steps")
    s.pop("workers", None)
    s["collision"] = LT[s.get("collision", 0)]
    if s.get("geometry") == "sphere48":
        s["geometry"] = SPHERE_RAW
    cfg = dlb.CaseConfig(**s)
    setup = {"tgv": dlb.init_tgv, "cavity": dlb.init_cavity, "porous": dlb.init_porous}[cfg.kind](cfg)
    return setup, bits, steps


def run_product(spec, slabs=1, arith="exact", steps=None):
    setup, bits, nsteps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, slabs=slabs, arith=arith)
    run.advance(nsteps if steps is None else steps)
    return run.gather_populations(), run


def raw_rel(a, b, q=19):
    w = descriptor(q)[1]
    n = a.size // q
    return np.max(np.abs(a - b).reshape(q, n) / (np.abs(b).reshape(q, n) + w[:, None]))


def macro(pops, q=19, fluid=None):
    """rho, u on fluid (Collide) cells; wall cells carry no macroscopic state
    (gather_macroscopic reports rho = 1, u = 0 / u_wall there, multiblock.cpp:464-479)."""
    c = descriptor(q)[0].astype(float)
    f = pops.reshape(q, -1)
    if fluid is not None:
        f = f[:, fluid]
    rho = 1.0 + f.sum(0)
    return rho, (c.T @ f) / rho


def fluid_mask(spec):
    setup, _, _ = product_setup(spec)
    kinds = np.asarray([ch.links[-1].type in (LinkType.BGK, LinkType.TRT, LinkType.RR)
                        for ch in setup.chains])
    idx = setup.chain_index
    if np.isscalar(idx):
        return None
    return kinds[idx].reshape(-1)


@pytest.mark.parametrize("name", list(CASES))
def test_exact_mode_bit_identical_to_reference(golden, name):
    """Every golden case, incl. config 1 at full size (cavity 64^3 BGK fp64,
    1000 steps), config 3/5 reduced and config 4 on a seeded sphere pack."""
    got, run = run_product(CASES[name])
    g = golden[name]
    assert np.array_equal(got[g["sample_index"]], np.asarray(g["sample"])), run.kernel_name()
    assert canonical_hash(got) == g["sha256"], run.kernel_name()


@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "cavity32_trt_f32", "tgv32_rr_f32", "plates16_trt_vel_f64"])
def test_exact_mode_vs_oracle_live(oracle, name):
    from golden_cases import make_case
    spec = CASES[name]
    got, _ = run_product(spec)
    want = oracle.run_case(make_case(spec), np.float64 if spec["bits"] == 64 else np.float32,
                           spec["steps"]).astype(np.float64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["tgv32_rr_f64", "cavity24_rr_f64", "tgv32_trt_f64", "sphere48_trt_f64_c4"])
def test_fast_mode_fp64_within_1e12(golden, oracle, name):
    from golden_cases import make_case
    spec = CASES[name]
    got, run = run_product(spec, arith="fast")
    want = oracle.run_case(make_case(spec), np.float64, spec["steps"])
    assert raw_rel(got, want) <= 1e-12
    assert "fast" in run.kernel_name()


@pytest.mark.parametrize("name", ["tgv128_bgk_f32_c5", "cavity32_trt_f32", "plates16_trt_pres_f32"])
def test_fast_mode_fp32_bounds(oracle, name):
    from golden_cases import make_case
    spec = CASES[name]
    got, _ = run_product(spec, arith="fast")
    want = oracle.run_case(make_case(spec), np.float32, spec["steps"]).astype(np.float64)
    assert raw_rel(got, want) <= 5e-5
    fl = fluid_mask(spec)
    r1, u1 = macro(got, fluid=fl)
    r0, u0 = macro(want, fluid=fl)
    assert np.max(np.abs(r1 - r0)) <= 1e-5 and np.max(np.abs(u1 - u0)) <= 1e-5


# ---------------------------------------------------------------- D3Q27 (config 2)
def q27_case(L, collision, bits, Re=1600.0, Ma=0.2):
    return dict(kind="tgv", L=L, Re=Re, Ma=Ma, collision=collision, q=27, bits=bits)


@pytest.mark.parametrize("collision,bits", [(RR, 64), (RR, 32), (BGK, 64), (TRT, 64)])
def test_d3q27_exact_bit_identical_to_oracle(oracle, collision, bits):
    spec = q27_case(24, collision, bits)
    steps = 30
    got, run = run_product(dict(spec, steps=steps))
    oc = Case(kind="tgv", L=24, Re=1600.0, Ma=0.2, collision=collision, q=27)
    want = oracle.run_case(oc, np.float64 if bits == 64 else np.float32, steps).astype(np.float64)
    assert np.array_equal(got, want), run.kernel_name()


def test_d3q27_rr_fast_fp64_within_1e12(oracle):
    got, _ = run_product(dict(q27_case(32, RR, 64), steps=40), arith="fast")
    want = oracle.run_case(Case(kind="tgv", L=32, Re=1600.0, Ma=0.2, collision=RR, q=27), np.float64, 40)
    assert raw_rel(got, want, 27) <= 1e-12


def test_d3q27_cavity_rr(oracle):
    spec = dict(kind="cavity", L=20, Re=400.0, Ma=0.1, collision=RR, q=27, bits=64, steps=60)
    got, _ = run_product(spec)
    want = oracle.run_case(Case(kind="cavity", L=20, Re=400.0, Ma=0.1, collision=RR, q=27), np.float64, 60)
    assert np.array_equal(got, want)


# ---------------------------------------------------------------- decomposition
@pytest.mark.parametrize("name,slabs", [("tgv16_bgk_f64", 2), ("tgv16_bgk_f64", 3), ("cavity32_trt_f32", 4),
                                        ("plates16_trt_vel_f64", 2), ("tgv32_rr_f32", 5)])
def test_zslab_decomposition_bit_identical(golden, name, slabs):
    """G z-slabs with the fused peer-memory halo push (here all on one GPU, each
    slab on its own stream with the flag protocol) == the single-slab result ==
    the reference (test_multiblock.cpp:234-256)."""
    got, run = run_product(CASES[name], slabs=slabs)
    assert canonical_hash(got) == golden[name]["sha256"]


def test_zslab_d3q27(oracle):
    spec = dict(q27_case(20, RR, 64), steps=25)
    a, _ = run_product(spec, slabs=1)
    b, _ = run_product(spec, slabs=3)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- API behaviour
def test_dispatch_error_before_any_write():
    """accelerated_lattice.cpp:161-181 / test_accelerated.cpp:223-244: a present
    tag outside the dispatch set fails the step and names the chain; no cell is
    touched."""
    cfg = dlb.CaseConfig(kind="cavity", L=16, Re=100.0, Ma=0.1)
    setup = dlb.init_cavity(cfg)
    reg = dlb.DynamicsRegistry()
    run = dlb.build_run(setup, reg, precision=64)
    run.advance(3)
    before = run.gather_populations()
    run.set_dispatch(dlb.DispatchSet.from_strings(reg, ["COLL_BGK", "BounceBack"]))
    with pytest.raises(dlb.DispatchError) as e:
        run.advance(1)
    assert e.value.chain_name == "MovingBounceBack"
    assert np.array_equal(run.gather_populations(), before)
    run.set_dispatch(dlb.DispatchSet.all_of(reg))
    run.advance(1)


def test_untagged_cell_dispatch_error():
    reg = dlb.DynamicsRegistry()
    s = reg.register_chain(dlb.make_collision_chain(LinkType.BGK, dlb.CollisionParams(omega=1.2)))
    run = dlb.DeviceRun((8, 8, 8), (1, 1, 1), reg)
    slots = np.full((8, 8, 8), s, np.int32)
    slots[3, 4, 5] = -1
    run.fill_slots(slots)
    run.fill_state()
    with pytest.raises(dlb.DispatchError) as e:
        run.advance(1)
    assert "<untagged cell>" in str(e.value)


def test_upload_download_roundtrip_and_hybrid(oracle):
    """Mirror-style hybrid execution (test_accelerated.cpp:170-186): 50 oracle
    steps, upload, 50 device steps == 100 oracle steps."""
    case = Case(kind="tgv", L=12, Re=8.0, Ma=0.1, collision=TRT)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    full = oracle.step(19, dims, per, rec, slot, f.copy(), 100)
    half = oracle.step(19, dims, per, rec, slot, f.copy(), 50)
    setup, _, _ = product_setup(dict(kind="tgv", L=12, Re=8.0, Ma=0.1, collision=TRT, bits=64, steps=0))
    run = dlb.build_run(setup, precision=64)
    run.upload_populations(half)
    assert np.array_equal(run.gather_populations(), half)
    run.advance(50)
    assert np.array_equal(run.gather_populations(), full)


def test_host_block_collide_and_stream_dropin(oracle):
    """dlb_collide_and_stream on a host AcceleratedBlock (envelope refreshed by
    the caller as refresh_envelope_periodic does) == the oracle step."""
    case = Case(kind="tgv", L=10, Re=50.0, Ma=0.1, collision=BGK)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    want = oracle.step(19, dims, per, rec, slot, f.copy(), 3)
    reg = dlb.DynamicsRegistry()
    cfg = dlb.CaseConfig(kind="tgv", L=10, Re=50.0, Ma=0.1)
    s = reg.register_chain(dlb.init_tgv(cfg).chains[0])
    n = 10
    blk = np.zeros((19, n + 2, n + 2, n + 2))
    blk[:, 1:-1, 1:-1, 1:-1] = f.reshape(19, n, n, n)
    tag = np.full((n + 2,) * 3, -1, np.int32)
    tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(s)
    pidx = np.where(tag >= 0, s, -1).astype(np.int32)
    for _ in range(3):
        dlb.refresh_envelope_periodic(blk, (1, 1, 1))
        dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet.all_of(reg))
    assert np.array_equal(blk[:, 1:-1, 1:-1, 1:-1].reshape(-1), want)
    with pytest.raises(dlb.DispatchError):
        dlb.collide_and_stream(reg, blk, tag, pidx, dlb.DispatchSet())
    # the same through page-locked host memory (zero-copy PCIe path)
    import ctypes as C
    from paper_2506_09242_b200 import _capi
    p = C.c_void_p()
    _capi.check(_capi.lib().dlb_host_alloc(blk.nbytes, C.byref(p)))
    try:
        pin = np.ctypeslib.as_array((C.c_uint8 * blk.nbytes).from_address(p.value)).view(np.float64).reshape(blk.shape)
        pin[:] = 0
        pin[:, 1:-1, 1:-1, 1:-1] = f.reshape(19, n, n, n)
        for _ in range(3):
            dlb.refresh_envelope_periodic(pin, (1, 1, 1))
            dlb.collide_and_stream(reg, pin, tag, pidx, dlb.DispatchSet.all_of(reg))
        assert np.array_equal(pin[:, 1:-1, 1:-1, 1:-1].reshape(-1), want)
    finally:
        _capi.lib().dlb_host_free(p)


def test_host_block_speculative_pipeline(oracle):
    """Pinned block, cached device lattice: the copies + step start while the
    eager tag scan runs. A dispatch error must still leave the block untouched,
    and a param_index change must recompute with the new slots."""
    import ctypes as C
    from paper_2506_09242_b200 import _capi
    n = 16
    case = Case(kind="cavity", L=n, Re=100.0, Ma=0.1, collision=TRT)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    bulk_only = np.zeros_like(slot)
    want = oracle.step(19, dims, per, rec, slot, f.copy(), 2)
    want = oracle.step(19, dims, per, rec, bulk_only, want, 1)   # param_index changed
    want = oracle.step(19, dims, per, rec, slot, want, 1)        # and back
    reg = dlb.DynamicsRegistry()
    setup = dlb.init_cavity(dlb.CaseConfig(kind="cavity", L=n, Re=100.0, Ma=0.1, collision=LinkType.TRT))
    slots = np.asarray([reg.register_chain(ch) for ch in setup.chains], np.int32)

    def tags_of(idx):
        tag = np.full((n + 2,) * 3, -1, np.int32)
        pidx = np.full((n + 2,) * 3, -1, np.int32)
        pidx[1:-1, 1:-1, 1:-1] = slots[idx]
        tag[1:-1, 1:-1, 1:-1] = np.vectorize(reg.tag_of_slot)(slots[idx])
        return tag, pidx
    real, bulk = tags_of(setup.chain_index), tags_of(np.zeros_like(setup.chain_index))
    p = C.c_void_p()
    nbytes = 19 * (n + 2) ** 3 * 8
    _capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
    try:
        pin = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(np.float64)
        pin = pin.reshape(19, n + 2, n + 2, n + 2)
        pin[:] = 0
        pin[:, 1:-1, 1:-1, 1:-1] = f.reshape(19, n, n, n)
        alld = dlb.DispatchSet.all_of(reg)
        for _ in range(2):
            dlb.collide_and_stream(reg, pin, *real, alld)
        before = pin.copy()
        with pytest.raises(dlb.DispatchError):  # speculative start, then the verdict
            dlb.collide_and_stream(reg, pin, *real, dlb.DispatchSet.from_strings(reg, [setup.chains[0].chain_string()]))
        assert np.array_equal(pin, before)
        dlb.collide_and_stream(reg, pin, *bulk, alld)
        dlb.collide_and_stream(reg, pin, *real, alld)
        assert np.array_equal(pin[:, 1:-1, 1:-1, 1:-1].reshape(-1), want)
    finally:
        _capi.lib().dlb_host_free(p)


def test_mass_conservation_long_run():
    """Periodic TGV: total mass drift <= 1e-12 relative over 1000 steps (acceptance.cpp:133-175)."""
    setup, _, _ = product_setup(dict(kind="tgv", L=32, Re=100.0, Ma=0.1, collision=BGK, bits=64, steps=0))
    run = dlb.build_run(setup, precision=64)
    m0 = run.gather_populations().sum()
    run.advance(1000)
    m1 = run.gather_populations().sum()
    n = 32 ** 3
    assert abs((n + m1) - (n + m0)) / n <= 1e-12


# ---------------------------------------------------------------- AA pattern
@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "cavity32_trt_f32", "plates16_trt_vel_f64",
                                  "tgv32_rr_f32", "sphere48_trt_f64_c4", "cavity64_bgk_f64_c1"])
def test_aa_layout_bit_identical_to_reference(golden, name):
    """In-place AA streaming (one array, half the memory) reproduces the
    reference after the golden step count (canonical state recovered from the
    even / odd layout on download)."""
    setup, bits, steps = product_setup(CASES[name])
    run = dlb.build_run(setup, precision=bits, layout="aa")
    run.advance(steps)
    assert canonical_hash(run.gather_populations()) == golden[name]["sha256"], run.kernel_name()
    assert "k_aa" in run.kernel_name()


@pytest.mark.parametrize("spec,steps", [
    (dict(kind="tgv", L=12, Re=50.0, Ma=0.1, collision=TRT, bits=64), 7),
    (dict(kind="cavity", L=18, Re=100.0, Ma=0.1, collision=BGK, bits=64), 13),
    (dict(kind="porous", L=12, Ma=0.01, collision=TRT, bits=32, plate_layers=4, upstream=3,
          downstream=3, drive="pressure"), 9),
    (dict(kind="tgv", L=14, Re=400.0, Ma=0.2, collision=RR, q=27, bits=64), 5),
])
def test_aa_odd_and_even_counts_vs_oracle(oracle, spec, steps):
    from golden_cases import make_case
    setup, bits, _ = product_setup(dict(spec, steps=0))
    run = dlb.build_run(setup, precision=bits, layout="aa")
    case = make_case(dict(spec, steps=0))
    dt = np.float64 if bits == 64 else np.float32
    f = oracle.initial_state(case, dt)
    dims, per, rec, slot = case.setup()
    for chunk in (1, steps - 1, 1, 2):  # stop at odd and even counts, download each time
        run.advance(chunk)
        oracle.step(case.q, dims, per, rec, slot, f, chunk)
        assert np.array_equal(run.gather_populations(), f.astype(np.float64))


def test_aa_upload_mid_run(oracle):
    case = Case(kind="tgv", L=10, Re=20.0, Ma=0.1, collision=BGK)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    oracle.step(19, dims, per, rec, slot, f, 3)
    setup, _, _ = product_setup(dict(kind="tgv", L=10, Re=20.0, Ma=0.1, collision=BGK, bits=64, steps=0))
    run = dlb.build_run(setup, precision=64, layout="aa")
    run.advance(1)  # leave the even layout, then overwrite the state
    run.upload_populations(f)
    run.advance(5)
    oracle.step(19, dims, per, rec, slot, f, 5)
    assert np.array_equal(run.gather_populations(), f)


# ---------------------------------------------------------------- masked porous variant
@pytest.mark.parametrize("name", ["sphere48_trt_f64_c4", "plates16_trt_vel_f64", "plates16_rr_vel_f64"])
def test_sparse_lists_fluid_cells_bit_identical(oracle, name):
    """Skipping NoDynamics cells (no loads / stores) leaves every Collide-kind
    cell bit-identical to the reference trajectory."""
    from golden_cases import make_case
    spec = CASES[name]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, sparse_lists=True)
    run.advance(steps)
    got = run.gather_populations().reshape(19, -1)
    want = oracle.run_case(make_case(spec), np.float64, steps).reshape(19, -1)
    fl = fluid_mask(spec)
    assert np.array_equal(got[:, fl], want[:, fl])
    assert "k_list" in run.kernel_name()  # single slab -> kind-sorted sparse lists
    assert run.step_bytes() < 304 * run.num_cells()


@pytest.mark.parametrize("group_bytes", [8, 32, 64, 256])
@pytest.mark.parametrize("name", ["sphere48_trt_f64_c4", "plates16_trt_vel_f64", "plates16_rr_vel_f64"])
def test_masked_sweep_fluid_cells_bit_identical(oracle, name, group_bytes, monkeypatch):
    """Masked sweep: all-NoDynamics segments (1 .. 32 cells) are skipped, mixed
    segments run the dense update; Collide-kind cells stay bit-identical."""
    from golden_cases import make_case
    monkeypatch.setenv("DLB_SKIP_GROUP_BYTES", str(group_bytes))
    spec = CASES[name]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    run.advance(steps)
    got = run.gather_populations().reshape(19, -1)
    want = oracle.run_case(make_case(spec), np.float64, steps).reshape(19, -1)
    fl = fluid_mask(spec)
    assert np.array_equal(got[:, fl], want[:, fl])
    nod = np.asarray(setup.chain_index).reshape(-1) == 2
    if nod.any():
        # single slab -> compacted sweep (x2 cells per thread in fp64)
        assert "k_cmp" in run.kernel_name() or "k_seg" in run.kernel_name()
        assert run.step_bytes() < 304 * run.num_cells()
    # stores cover at least every Collide / wall cell (wall cells load only fluid-facing links)
    assert run.step_bytes() >= 152 * int((~nod).sum())  # every listed cell stores its q links


@pytest.mark.parametrize("cpt", ["1", "2"])
def test_segment_sweep_cells_per_thread(oracle, cpt, monkeypatch):
    """k_seg with one and two cells per thread: Collide-kind cells bit-identical."""
    from golden_cases import make_case
    monkeypatch.setenv("DLB_SEG_CPT", cpt)
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    assert f",x{cpt}>" in run.kernel_name()
    run.advance(steps)
    got = run.gather_populations().reshape(19, -1)
    want = oracle.run_case(make_case(spec), np.float64, steps).reshape(19, -1)
    fl = fluid_mask(spec)
    assert np.array_equal(got[:, fl], want[:, fl])


def test_masked_dense_sweep_fluid_cells_bit_identical(oracle, monkeypatch):
    """The uncompacted masked sweep (warp ballot over x-aligned segments)."""
    from golden_cases import make_case
    monkeypatch.setenv("DLB_MASKED_COMPACT", "0")
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    run.advance(steps)
    got = run.gather_populations().reshape(19, -1)
    want = oracle.run_case(make_case(spec), np.float64, steps).reshape(19, -1)
    fl = fluid_mask(spec)
    assert np.array_equal(got[:, fl], want[:, fl])
    assert "SKIP" in run.kernel_name()


def test_skip_nodynamics_zslabs_masked_dense(oracle):
    """With z-slabs the masked dense sweep (KM_SKIP) is used instead of lists."""
    from golden_cases import make_case
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True, slabs=3)
    run.advance(60)
    got = run.gather_populations().reshape(19, -1)
    want = oracle.run_case(make_case(spec), np.float64, 60).reshape(19, -1)
    fl = fluid_mask(spec)
    assert np.array_equal(got[:, fl], want[:, fl])
    assert "SKIP" in run.kernel_name()


# ---------------------------------------------------------------- checksums / full size
def test_checksum_matches_oracle():
    from pyoracle import Oracle, canonical_checksum
    case = Case(kind="cavity", L=24, Re=400.0, Ma=0.1, collision=TRT)
    want = canonical_checksum(Oracle().run_case(case, np.float32, 40).astype(np.float64))
    setup, _, _ = product_setup(dict(kind="cavity", L=24, Re=400.0, Ma=0.1, collision=TRT, bits=32, steps=0))
    for layout, slabs in (("twopop", 1), ("aa", 1), ("twopop", 3)):
        run = dlb.build_run(setup, precision=32, layout=layout, slabs=slabs)
        run.advance(40)
        assert run.checksum() == want, (layout, slabs)


@pytest.mark.parametrize("layout,slabs", [("twopop", 1), ("twopop", 4), ("aa", 1), ("aa", 2)])
def test_full_size_config3_matches_reference_checksum(layout, slabs):
    """Config 3 at its full per-GPU size (cavity 512^3 D3Q19 TRT fp32): the
    device state after the reference's step count has the reference's exact
    checksum (tests/golden/golden_full.json, made from oracle/_ref) -- also as
    linked z-slabs (the walls and the lid land in different slabs) and in the
    AA layout."""
    import json
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_full.json")
    g = json.load(open(path))["cavity512_trt_f32_c3_full"]
    spec = dict(g["spec"])
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, layout=layout, slabs=slabs)
    run.advance(steps)
    assert run.checksum() == [int(v) for v in g["checksum"]]


def test_full_size_config5_layout_and_decomposition_invariance():
    """Config 5 at full size (TGV D3Q19 BGK fp32 1024^3, 169 GB two-population):
    two-population, AA in place, and 2 z-slabs of either give identical checksums."""
    cfg = dlb.CaseConfig(kind="tgv", L=1024, Re=1600.0, Ma=0.2)
    sums = []
    for layout, slabs in (("twopop", 1), ("aa", 1), ("twopop", 2), ("aa", 2)):
        run = dlb.build_run(dlb.init_tgv(cfg), precision=32, layout=layout, slabs=slabs)
        run.advance(5)
        sums.append(run.checksum())
        del run
    assert sums[0] == sums[1] == sums[2] == sums[3]


@pytest.mark.parametrize("layout", ["twopop", "aa"])
def test_graph_replay_any_parity(oracle, layout):
    """Steps replay as a captured 2-step CUDA graph; odd chunk sizes and
    restarts at either parity must not change the trajectory."""
    case = Case(kind="cavity", L=20, Re=200.0, Ma=0.1, collision=TRT)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float64)
    setup, _, _ = product_setup(dict(kind="cavity", L=20, Re=200.0, Ma=0.1, collision=TRT, bits=64, steps=0))
    run = dlb.build_run(setup, precision=64, layout=layout)
    for chunk in (1, 9, 4, 1, 1, 17, 6):
        run.advance(chunk)
        oracle.step(19, dims, per, rec, slot, f, chunk)
        assert np.array_equal(run.gather_populations(), f), chunk


# ---------------------------------------------------------------- macroscopic fields / dumps
@pytest.mark.parametrize("name,layout", [("cavity32_trt_f32", "twopop"), ("plates16_trt_vel_f64", "aa"),
                                         ("tgv24_smag_bgk_f64", "twopop")])
def test_gather_macroscopic_matches_reference(reference, name, layout):
    from golden_cases import make_case
    spec = CASES[name]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, layout=layout)
    run.advance(steps)
    got = run.gather_macroscopic()
    want = reference.macroscopic(make_case(spec), bits, steps)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "cavity32_trt_f32"])
def test_field_dump_bytes_match_reference(reference, tmp_path, name):
    """DOLB1 dump written from the device state is byte-identical to the
    reference's write_field_dump of the same run (accelerated_lattice.cpp:313-341)."""
    from golden_cases import make_case
    spec = CASES[name]
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits)
    run.advance(steps)
    mine, ref = tmp_path / "mine.dolb", tmp_path / "ref.dolb"
    run.write_field_dump(str(mine))
    reference.dump(make_case(spec), bits, steps, str(ref))
    assert mine.read_bytes() == ref.read_bytes()
    dims, prec, data = dlb.read_field_dump(str(mine))
    assert dims == setup.dims and prec == bits // 8
    assert np.array_equal(data, run.gather_populations())



# ---------------------------------------------------------------- TMA vs plain-load kernels
@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "tgv12_bgk_f32", "cavity32_trt_f32", "cavity64_bgk_f64_c1",
                                  "tgv128_bgk_f32_c5", "cavity128_trt_f32_c3"])
def test_tma_and_plain_kernels_bit_identical_to_reference(golden, name):
    """The TMA-staged kernel (opt-in) and the default plain-load kernel both
    reproduce the reference bit for bit."""
    setup, bits, steps = product_setup(CASES[name])
    names = []
    for tma in (True, False):
        run = dlb.build_run(setup, precision=bits, tma=tma)
        run.advance(steps)
        assert canonical_hash(run.gather_populations()) == golden[name]["sha256"], run.kernel_name()
        names.append(run.kernel_name())
    assert "k_tma" in names[0] and "k_pull" in names[1]  # k_tmarow (row-staged) or k_tma (box-tiled)


def test_tma_d3q27_rr(oracle):
    spec = dict(q27_case(24, RR, 64), steps=12)
    setup, bits, steps = product_setup(spec)
    run = dlb.build_run(setup, precision=bits, tma=True)
    run.advance(steps)
    got = run.gather_populations()
    want = oracle.run_case(Case(kind="tgv", L=24, Re=1600.0, Ma=0.2, collision=RR, q=27), np.float64, 12)
    assert np.array_equal(got, want)
    assert "k_tma" in run.kernel_name()


def test_tma_envelope_after_upload_and_odd_counts(oracle):
    """The periodic envelope images are re-primed after an upload and kept
    current across single steps and graph replays."""
    case = Case(kind="tgv", L=20, Re=50.0, Ma=0.1, collision=TRT)
    dims, per, rec, slot = case.setup()
    f = oracle.initial_state(case, np.float32)
    setup, _, _ = product_setup(dict(kind="tgv", L=20, Re=50.0, Ma=0.1, collision=TRT, bits=32, steps=0))
    run = dlb.build_run(setup, precision=32, tma=True)
    assert "k_tma" in run.kernel_name()
    run.advance(3)
    run.upload_populations(f.astype(np.float64))
    for chunk in (1, 6, 1, 9):
        run.advance(chunk)
        oracle.step(19, dims, per, rec, slot, f, chunk)
        assert np.array_equal(run.gather_populations(), f.astype(np.float64)), chunk


@pytest.mark.parametrize("bits", [64, 32])
def test_fluid_segment_sweep_interleaved_reads(oracle, bits, monkeypatch):
    """Fluid-segment sweep (k_segbb): wall cells outside the fluid segments skip
    their steps and are brought up to date lazily whenever the state is read.
    Chunked advances (graph and single-step paths) with gathers, checksums and
    macroscopic fields in between: every non-NoDynamics cell -- collision and
    bounce-back -- bit-identical to the oracle at every read, and equal to the
    plain masked sweep (the default)."""
    from golden_cases import make_case
    spec = dict(CASES["sphere48_trt_f64_c4"], bits=bits)
    setup, _, _ = product_setup(spec)
    case = make_case(spec)
    dims, per, rec, slot = case.setup()
    dt = np.float64 if bits == 64 else np.float32
    f = oracle.initial_state(case, dt)
    monkeypatch.setenv("DLB_FLUID_SEGMENTS", "1")
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    assert "k_segbb" in run.kernel_name()
    monkeypatch.setenv("DLB_FLUID_SEGMENTS", "0")
    ref = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    assert "k_segbb" not in ref.kernel_name()
    active = np.asarray(setup.chain_index).reshape(-1) != 2
    for chunk in (1, 1, 5, 2, 7, 1, 12):
        run.advance(chunk)
        ref.advance(chunk)
        oracle.step(19, dims, per, rec, slot, f, chunk)
        got = run.gather_populations().reshape(19, -1)
        want = np.asarray(f, np.float64).reshape(19, -1)
        assert np.array_equal(got[:, active], want[:, active]), chunk
        assert run.checksum(active_only=True) == ref.checksum(active_only=True)
        assert all(np.array_equal(a, b) for a, b in zip(run.gather_macroscopic(), ref.gather_macroscopic()))
    # fewer bytes per step than the masked sweep it replaces
    assert run.step_bytes() < ref.step_bytes()


def test_fluid_segment_sweep_restarts_after_upload(oracle, monkeypatch):
    """An upload (or fill) makes the next step a full masked step again (the
    two buffers are not ping-pong current any more)."""
    from golden_cases import make_case
    monkeypatch.setenv("DLB_FLUID_SEGMENTS", "1")
    spec = CASES["sphere48_trt_f64_c4"]
    setup, bits, _ = product_setup(spec)
    case = make_case(spec)
    dims, per, rec, slot = case.setup()
    run = dlb.build_run(setup, precision=bits, skip_nodynamics=True)
    assert "k_segbb" in run.kernel_name()
    run.advance(9)
    f = oracle.initial_state(case, np.float64)
    oracle.step(19, dims, per, rec, slot, f, 3)
    run.upload_populations(f)
    run.advance(6)
    oracle.step(19, dims, per, rec, slot, f, 6)
    active = np.asarray(setup.chain_index).reshape(-1) != 2
    got = run.gather_populations().reshape(19, -1)
    assert np.array_equal(got[:, active], f.reshape(19, -1)[:, active])


# ---------------------------------------------------------------- 128-bit vectorised sweep
@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "cavity32_trt_f32", "cavity64_bgk_f64_c1"])
def test_vectorised_sweep_bit_identical_to_reference(golden, name, monkeypatch):
    """k_vec (DLB_VEC=1): one 128-bit load / store per direction and thread
    (4 fp32 or 2 fp64 cells), +-1 x shifts through warp shuffles; same per-cell
    arithmetic as k_pull, so the reference's goldens hold bit for bit."""
    monkeypatch.setenv("DLB_VEC", "1")
    setup, bits, steps = product_setup(CASES[name])
    run = dlb.build_run(setup, precision=bits)
    assert "k_vec" in run.kernel_name(), run.kernel_name()
    run.advance(steps)
    assert canonical_hash(run.gather_populations()) == golden[name]["sha256"]


@pytest.mark.parametrize("dims,periodic", [((36, 7, 5), (1, 1, 1)), ((40, 9, 6), (0, 1, 0)), ((8, 3, 3), (1, 0, 1))])
@pytest.mark.parametrize("bits", [32, 64])
def test_vectorised_sweep_ragged_vs_oracle(oracle, dims, periodic, bits, monkeypatch):
    """Rows of 2-10 vectors, partial warps and blocks, periodic / walled x."""
    monkeypatch.setenv("DLB_VEC", "1")
    reg = dlb.DynamicsRegistry()
    p = dlb.CollisionParams()
    p.set_trt(1.3, 0.25)
    s = reg.register_chain(dlb.make_collision_chain(LinkType.TRT, p))
    run = dlb.DeviceRun(dims, periodic, reg, precision=bits)
    run.fill_slots(s)
    rng = np.random.default_rng(sum(dims) + bits)
    n = dims[0] * dims[1] * dims[2]
    f0 = rng.normal(0.0, 1e-3, 19 * n)
    if bits == 32:
        f0 = f0.astype(np.float32).astype(np.float64)
    run.upload_populations(f0)
    assert "k_vec" in run.kernel_name()
    run.advance(5)
    monkeypatch.setenv("DLB_VEC", "0")
    ref2 = dlb.DeviceRun(dims, periodic, reg, precision=bits)
    ref2.fill_slots(s)
    ref2.upload_populations(f0)
    ref2.advance(5)
    assert "k_vec" not in ref2.kernel_name()
    assert np.array_equal(run.gather_populations(), ref2.gather_populations())
