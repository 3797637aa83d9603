"""GPU-resident diagnostics: the runner's sampling step
(proj/src/runner.cpp:346-448) computed from the resident state must equal the
reference's host computation (diag::tree_sum / kinetic_energy / vorticity_fd8 /
enstrophy / permeability, proj/src/diagnostics.cpp:10-131) BIT FOR BIT.

CPU part: the split tree reduction (plan per segment + combine) against the
reference's diag::tree_sum on random sequences and segmentations, and the
golden sampling values against the live reference. GPU part (-m gpu): device
values against tests/golden/golden_diag.json and the live reference, for
single slabs, z-slab decompositions, the AA layout and forced chunking."""
import ctypes as C
import json
import os
import struct

import numpy as np
import pytest

from golden_cases import CASES, DIAG_CASES, make_case
from paper_2506_09242_b200 import _capi

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_DIAG = os.path.join(HERE, "golden", "golden_diag.json")


def bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]


def dlb_tree_sum(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, np.float64)
    out = C.c_double()
    _capi.check(_capi.lib().dlb_tree_sum(v.ctypes.data if v.size else None, v.size, C.byref(out)))
    return out.value


def plan(n_total, a, b):
    n = C.c_size_t()
    _capi.check(_capi.lib().dlb_tree_plan(n_total, a, b, None, 0, C.byref(n)))
    buf = (_capi.TreePart * max(n.value, 1))()
    _capi.check(_capi.lib().dlb_tree_plan(n_total, a, b, buf, n.value, C.byref(n)))
    return list(buf[:n.value])


def combine(n_total, parts):
    arr = (_capi.TreePart * max(len(parts), 1))(*parts)
    out = C.c_double()
    st = _capi.lib().dlb_tree_combine(n_total, arr, len(parts), C.byref(out))
    return st, out.value


def spread(rng, n):
    """Values spanning many magnitudes and both signs (association matters)."""
    return rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, n)


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 16, 17, 100, 1023, 4097, 100003])
def test_tree_sum_matches_reference(reference, n):
    rng = np.random.default_rng(n)
    v = spread(rng, n)
    assert bits(dlb_tree_sum(v)) == bits(reference.tree_sum(v))


@pytest.mark.parametrize("seed", range(12))
def test_split_tree_reduction_bit_identical(reference, seed):
    """Any segmentation (slabs, device chunks) -> parts -> combine == tree_sum."""
    rng = np.random.default_rng(100 + seed)
    n_total = int(rng.integers(1, 50000)) if seed else 9
    v = spread(rng, n_total)
    ncut = int(rng.integers(0, 12))
    cuts = sorted(set([0, n_total] + rng.integers(0, n_total + 1, ncut).tolist()))
    parts = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        for p in plan(n_total, a, b):
            assert a <= p.lo and p.lo + max(p.len, 1) <= b
            p.value = dlb_tree_sum(v[p.lo:p.lo + p.len]) if p.len else v[p.lo]
            parts.append(p)
    rng.shuffle(parts)
    st, got = combine(n_total, parts)
    assert st == 0
    assert bits(got) == bits(reference.tree_sum(v))


def test_tree_combine_reports_missing_parts():
    parts = plan(1000, 0, 400)  # the rest of the sequence is missing
    for p in parts:
        p.value = 1.0
    st, _ = combine(1000, parts)
    assert st == 1  # DLB_ERROR_INVALID_ARGUMENT
    assert b"no part covers" in _capi.lib().dlb_last_error()


def test_tree_plan_rejects_bad_segments():
    n = C.c_size_t()
    assert _capi.lib().dlb_tree_plan(10, 5, 11, None, 0, C.byref(n)) == 1
    assert _capi.lib().dlb_tree_plan(10, 6, 5, None, 0, C.byref(n)) == 1


def load_golden():
    with open(GOLDEN_DIAG) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["tgv16_bgk_f64", "tgv12_bgk_f32", "cavity24_rr_f64", "plates16_trt_vel_f64"])
def test_golden_diag_matches_live_reference(reference, name):
    """The committed goldens are the reference's own numbers (pins the fixture)."""
    g = load_golden()[name]
    spec = CASES[name]
    vals = reference.sample(make_case(spec), spec["bits"], *g["steps"])
    for k, hx in g["values"].items():
        assert bits(vals[k]) == bits(float.fromhex(hx)), k


# ---------------------------------------------------------------------------
# device side

def product_run(name, slabs=1, layout="twopop"):
    import paper_2506_09242_b200 as dlb
    from test_gpu_parity import product_setup
    spec = CASES[name]
    setup, bits_, _ = product_setup(spec)
    run = dlb.build_run(setup, precision=bits_, slabs=slabs, layout=layout)
    return run, setup


def device_sample(name, slabs=1, layout="twopop"):
    """The runner's sampling step on the device: snapshot after steps_a, all
    values after steps_a + steps_b."""
    import paper_2506_09242_b200 as dlb
    spec = CASES[name]
    a, b = DIAG_CASES[name]
    run, setup = product_run(name, slabs, layout)
    run.advance(a)
    run.snapshot_velocity()
    run.advance(b)
    nn, dd = run.convergence_sums()
    out = {"k": run.kinetic_energy(), "eps": run.enstrophy(), "nn": nn, "dd": dd}
    if spec["kind"] == "porous":
        cfg = dlb.CaseConfig(**{k: v for k, v in product_cfg_kwargs(spec).items()})
        ex = run.porous_extras(setup.sample_begin, setup.sample_end, cfg.viscosity(),
                               aperture_mean=cfg.geometry == "plates")
    else:
        ex = [0.0] * 5
    out.update(zip(["k_perm", "ubar", "dp", "ux_in", "ux_out"], ex))
    return out


def product_cfg_kwargs(spec):
    from test_gpu_parity import LT
    from golden_cases import SPHERE_RAW
    s = dict(spec)
    for k in ("bits", "steps", "workers"):
        s.pop(k, None)
    s["collision"] = LT[s.get("collision", 0)]
    if s.get("geometry") == "sphere48":
        s["geometry"] = SPHERE_RAW
    return s


def assert_same(got, golden_values):
    bad = {k: (got[k], float.fromhex(h)) for k, h in golden_values.items() if bits(got[k]) != bits(float.fromhex(h))}
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(DIAG_CASES))
def test_device_sampling_bit_identical_to_reference(name):
    assert_same(device_sample(name), load_golden()[name]["values"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,slabs", [("tgv32_rr_f64", 3), ("cavity32_trt_f32", 2),
                                        ("plates16_trt_pres_f32", 2), ("tgv16_bgk_f64", 4)])
def test_device_sampling_zslabs(name, slabs):
    """Slabs reduce their own tree nodes; the enstrophy stencil reads 4 halo
    planes from the neighbours (tgv16 / 4 slabs: every slab is exactly 4 thick)."""
    assert_same(device_sample(name, slabs=slabs), load_golden()[name]["values"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tgv32_rr_f64", "cavity24_rr_f64", "sphere48_trt_f64_c4"])
def test_device_sampling_aa_layout(name):
    assert_same(device_sample(name, layout="aa"), load_golden()[name]["values"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tgv128_bgk_f32_c5", "sphere48_trt_f64_c4", "cavity32_trt_f32"])
def test_device_sampling_forced_chunks(name, monkeypatch):
    """A minimal scratch buffer forces 2-plane device chunks: many segment
    boundaries, leaves cut between chunks, compaction per chunk."""
    monkeypatch.setenv("DLB_DIAG_SCRATCH_BYTES", "1")
    assert_same(device_sample(name), load_golden()[name]["values"])


@pytest.mark.gpu
def test_device_sampling_live_reference(reference):
    """An extra case straight against the reference (not in the fixtures)."""
    spec = dict(CASES["plates16_bgk_pres_f64"])
    name = "plates16_bgk_pres_f64"
    DIAG_CASES_local = (60, 40)
    import paper_2506_09242_b200 as dlb
    run, setup = product_run(name)
    run.advance(DIAG_CASES_local[0])
    run.snapshot_velocity()
    run.advance(DIAG_CASES_local[1])
    nn, dd = run.convergence_sums()
    cfg = dlb.CaseConfig(**product_cfg_kwargs(spec))
    got = {"k": run.kinetic_energy(), "eps": run.enstrophy(), "nn": nn, "dd": dd}
    got.update(zip(["k_perm", "ubar", "dp", "ux_in", "ux_out"],
                   run.porous_extras(setup.sample_begin, setup.sample_end, cfg.viscosity(), True)))
    ref = reference.sample(make_case(spec), spec["bits"], *DIAG_CASES_local)
    assert_same(got, {k: float(v).hex() for k, v in ref.items()})


@pytest.mark.gpu
def test_velocity_planes_match_gather_macroscopic():
    run, _ = product_run("cavity24_rr_f64")
    run.advance(7)
    _, ux, uy, uz = run.gather_macroscopic()
    nx, ny, nz = run.dims
    planes = run.velocity_planes(3, 5)
    for c, u in enumerate((ux, uy, uz)):
        assert np.array_equal(planes[:, c], u.reshape(nz, ny, nx)[3:8])


@pytest.mark.gpu
def test_du_without_snapshot_is_an_error():
    import paper_2506_09242_b200 as dlb
    run, _ = product_run("tgv16_bgk_f64")
    with pytest.raises(dlb.DlbError):
        run.tree_reduce(_capi.Q_DU_NUM)


@pytest.mark.gpu
@pytest.mark.parametrize("name,fused", [("tgv16_bgk_f64", True), ("tgv12_bgk_f32", True), ("tgv32_rr_f64", True),
                                        ("tgv24_smag_trt_f32", True), ("tgv128_bgk_f32_c5", True),
                                        ("cavity64_bgk_f64_c1", True), ("cavity32_trt_f32", True),
                                        ("cavity24_rr_f64", True), ("plates16_trt_vel_f64", False)])
def test_fused_kinetic_energy_bit_identical(name, fused):
    """Fused collide + reduce (dlb_lattice_request_kinetic): the last step of
    the advance writes the per-cell kinetic energy, the reduction reads those
    values -- the same bits as the unfused sampling and the reference's
    diag::kinetic_energy. Regularized inlet / outlet lattices (fix-up lists)
    fall back to the unfused path."""
    a, b = DIAG_CASES[name]
    run, _ = product_run(name, 1, "twopop")
    run.advance(a)
    assert run.request_kinetic() == fused
    run.advance(b)
    k = run.kinetic_energy()
    assert bits(k) == bits(float.fromhex(load_golden()[name]["values"]["k"]))
    # the values belong to that state only: after one more step the reduction is unfused again
    run.advance(1)
    k1 = run.kinetic_energy()
    run2, _ = product_run(name, 1, "twopop")
    run2.advance(a + b + 1)
    assert bits(k1) == bits(run2.kinetic_energy())


@pytest.mark.gpu
def test_fused_kinetic_energy_unavailable_paths():
    """fast arithmetic, the AA layout and z-slabs have no fused variant."""
    name = "tgv16_bgk_f64"
    for kw in ({"layout": "aa"}, {"slabs": 2}):
        run, _ = product_run(name, kw.get("slabs", 1), kw.get("layout", "twopop"))
        assert not run.request_kinetic()
        run.advance(10)
        assert bits(run.kinetic_energy()) == bits(float.fromhex(load_golden()[name]["values"]["k"]))


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [64, 32])
def test_fused_kinetic_energy_d3q27(oracle, bits):
    """D3Q27 RR (config 2's lattice): fused kinetic energy equals the unfused reduction."""
    import numpy as np
    import paper_2506_09242_b200 as dlb
    cfg = dlb.CaseConfig(kind="tgv", L=24, Re=1600.0, Ma=0.2, collision=dlb.LinkType.RR, q=27)
    setup = dlb.init_tgv(cfg)
    a = dlb.build_run(setup, precision=bits)
    b = dlb.build_run(setup, precision=bits)
    a.advance(7)
    assert b.request_kinetic()
    b.advance(7)
    assert bits_(a.kinetic_energy()) == bits_(b.kinetic_energy())


def bits_(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]
