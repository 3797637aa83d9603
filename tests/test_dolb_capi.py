"""The reference's benchmark-level C interface (include/dolb.h) served by the
device runner: the assertions of proj/tests/test_capi.cpp:26-111 restated, the
reference's configuration errors and show_models output, and -- on the GPU --
dolb_run artefacts byte-identical to the reference's own dolb_run
(tests/golden/runner/, from tests/golden/make_runner_golden.py), manifest
replay (test_runner.cpp:120-125) and dispatch failures.
"""
import hashlib
import json
import os
import shutil

import pytest

from paper_2506_09242_b200.runner import CONFIG, DISPATCH, DOLB_LIB, INTERNAL, INVALID_ARGUMENT, Dolb, DolbError
from runner_cases import RUNNER_CASES, normalize_manifest, resolve_paths

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "runner")
REF_LIB = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "libdolb_ref.so")


def gpu_present() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="module")
def api():
    return Dolb()


# ------------------------------------------------------------------ CPU: C surface
def test_library_exports_every_dolb_h_symbol():
    import ctypes as C
    import re
    header = open(os.path.join(os.path.dirname(HERE), "include", "dolb.h")).read()
    declared = set(re.findall(r"DOLB_API\s+[\w\s\*]+?\b(dolb_\w+)\s*\(", header))
    assert len(declared) == 12, declared
    lib = C.CDLL(DOLB_LIB)  # the libdolb.so name the reference's callers link against
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing


def test_version_and_null_arguments(api):
    lib = api.lib
    assert "." in api.version()
    assert lib.dolb_config_load(None, b"x") == INVALID_ARGUMENT
    assert lib.dolb_config_set(None, b"a", b"b") == INVALID_ARGUMENT
    assert lib.dolb_run(None, None, None) == INVALID_ARGUMENT
    assert "null" in api.last_error()
    assert lib.dolb_show_models(None, None, 0, None) == INVALID_ARGUMENT
    assert lib.dolb_bytes_per_cell(32, None) == INVALID_ARGUMENT


def test_config_round_trip(api):
    import ctypes as C
    with api.config() as cfg:
        cfg.set("case.kind", "tgv")
        assert cfg.get("case.kind") == "tgv"
        buf = C.create_string_buffer(16)
        assert api.lib.dolb_config_get(cfg.handle, b"case.missing", buf, 16) == INVALID_ARGUMENT
        assert api.lib.dolb_config_get(cfg.handle, b"case.kind", buf, 2) == INVALID_ARGUMENT


def test_config_file_sections_comments_and_override(api, tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# comment\n[case]\nkind = cavity   # trailing\nL = 24\n\n[run]\ntmax = 5tc\n")
    with api.config() as cfg:
        cfg.set("case.L", "16")
        cfg.load(str(p))
        assert cfg.get("case.kind") == "cavity" and cfg.get("case.L") == "24" and cfg.get("run.tmax") == "5tc"
        cfg.set("case.L", "32")  # later set wins
        assert cfg.get("case.L") == "32"
    bad = tmp_path / "bad.cfg"
    bad.write_text("[case]\nno equals sign\n")
    with api.config() as cfg:
        with pytest.raises(DolbError) as e:
            cfg.load(str(bad))
        assert e.value.status == 3 and "without '='" in e.value.message
        with pytest.raises(DolbError) as e:
            cfg.load(str(tmp_path / "missing.cfg"))
        assert e.value.status == 3


# error texts of the reference's resolve / CaseConfig::validate (runner.cpp:151-267, cases.cpp:52-68)
CONFIG_ERRORS = [
    ({"case.kind": "vortex-street"}, 'unknown case "vortex-street"; valid cases: tgv, cavity, porous'),
    ({"case.collision": "mrt"}, 'unknown collision model "mrt"; valid models: bgk, trt, rr'),
    ({"case.precision": "f16"}, 'unknown precision "f16"; valid precisions: f32, f64'),
    ({"case.drive": "gravity", "case.kind": "porous", "case.geometry": "plates"},
     'unknown drive "gravity"; valid drives: velocity, pressure'),
    ({"run.tmax": "abc"}, 'cannot parse time specification "abc": use steps, "<N>tc" or "steady"'),
    ({"case.L": "4"}, "tgv requires L >= 8"),
    ({"case.kind": "cavity", "case.L": "8"}, "cavity requires L >= 16"),
    ({"case.kind": "porous"}, "porous case requires a geometry"),
    ({"case.Ma": "0.7"}, "Mach number must lie in (0, 0.5)"),
    ({"run.output_every": "0"}, "run.output_every must be >= 1"),
    ({"case.L": "x"}, 'config key case.L: "x" is not an integer'),
    ({"case.Re": "1e"}, 'config key case.Re: "1e" is not a number'),
    ({"run.reference_check": "maybe"}, 'config key run.reference_check: "maybe" is not a boolean'),
    ({"run.blocks": "1,2"}, "run.blocks needs three comma-separated counts"),
    ({"case.kind": "porous", "case.geometry": "g.raw"}, "voxel geometry needs case.voxel_dims"),
]


@pytest.mark.parametrize("values,message", CONFIG_ERRORS)
def test_configuration_errors_surface_with_reference_messages(api, values, message, tmp_path):
    with pytest.raises(DolbError) as e:
        api.run(dict(values, **{"run.out": str(tmp_path)}))
    assert e.value.status == CONFIG
    assert message in e.value.message


def test_missing_voxel_file_is_io_error(api, tmp_path):
    with pytest.raises(DolbError) as e:
        api.run({"case.kind": "porous", "case.geometry": str(tmp_path / "none.raw"), "case.voxel_dims": "4,4,4",
                 "run.out": str(tmp_path)})
    assert e.value.status == 3 and "cannot open voxel file" in e.value.message


def test_show_models_sizes_and_fills_the_buffer(api):
    import ctypes as C
    with api.config({"case.kind": "tgv", "case.L": "8", "case.Re": "8", "case.Ma": "0.1"}) as cfg:
        n = C.c_size_t()
        assert api.lib.dolb_show_models(cfg.handle, None, 0, C.byref(n)) == 0
        assert n.value == len("COLL_BGK\n") + 1
        buf = C.create_string_buffer(n.value)
        assert api.lib.dolb_show_models(cfg.handle, buf, n.value, None) == 0
        assert buf.value == b"COLL_BGK\n"
        tiny = C.create_string_buffer(4)
        assert api.lib.dolb_show_models(cfg.handle, tiny, 4, None) == INVALID_ARGUMENT


SHOW_CASES = [
    {"case.kind": "cavity", "case.L": "16", "case.collision": "trt"},
    {"case.kind": "porous", "case.geometry": "plates", "case.L": "20", "case.H": "6"},
    {"case.kind": "porous", "case.geometry": "plates", "case.L": "20", "case.drive": "pressure",
     "case.collision": "rr"},
    {"case.kind": "tgv", "case.smagorinsky": "0.1", "case.collision": "trt"},
    {"case.kind": "porous", "case.geometry": "@SPHERE", "case.voxel_dims": "48,48,48"},
]
SHOW_EXPECTED = [
    ["BounceBack", "COLL_TRT", "MovingBounceBack"],
    ["BounceBack", "Boundary_RegularizedVelocity_0_1__TRT", "Boundary_RegularizedVelocity_0_M1__TRT", "COLL_TRT"],
    ["BounceBack", "Boundary_RegularizedPressure_0_1__RR", "Boundary_RegularizedPressure_0_M1__RR", "COLL_RR"],
    ["LES_Smagorinsky|COLL_TRT"],
    ["BounceBack", "Boundary_RegularizedVelocity_0_1__TRT", "Boundary_RegularizedVelocity_0_M1__TRT", "COLL_TRT",
     "NoDynamics"],
]


@pytest.mark.parametrize("k", range(len(SHOW_CASES)))
def test_show_models_matches_reference(api, k):
    values = resolve_paths(SHOW_CASES[k], "unused")
    got = api.show_models(values)
    assert got == SHOW_EXPECTED[k]
    if os.path.exists(REF_LIB):  # the reference's own answer (no run, so no locale issue)
        assert Dolb(REF_LIB).show_models(values) == got


def test_performance_model_queries(api):
    assert api.bytes_per_cell(32) == 164
    assert api.bytes_per_cell(64) == 316
    with pytest.raises(DolbError) as e:
        api.bytes_per_cell(31)
    assert e.value.status == CONFIG
    assert abs(api.peak_glups("A100-SXM4-40GB", 32) - 9.481) <= 1e-3
    with pytest.raises(DolbError) as e:
        api.peak_glups("nonexistent", 32)
    assert e.value.status == CONFIG
    assert abs(api.memory_fraction("A100-SXM4-40GB", 64, 500) - 0.9875) <= 1e-4


def test_device_catalog_file(api, tmp_path):
    cat = tmp_path / "devices.txt"
    cat.write_text("# name GB/s GB\nB200 8000 180\n")
    assert abs(api.peak_glups("B200", 32, str(cat)) - 8000e9 / 164 / 1e9) < 1e-9
    assert abs(api.memory_fraction("B200", 32, 1024, str(cat)) - 164 * 1024 ** 3 / 180e9) < 1e-12


@pytest.mark.skipif(gpu_present(), reason="checks the no-GPU failure mode")
def test_run_without_gpu_fails_loudly(api, tmp_path):
    with pytest.raises(DolbError) as e:
        api.run({"case.kind": "tgv", "case.L": "8", "case.Re": "8", "case.Ma": "0.1", "run.tmax": "2",
                 "run.out": str(tmp_path)})
    assert e.value.status == INTERNAL


# ------------------------------------------------------------------ GPU: dolb_run
@pytest.mark.gpu
def test_tiny_run_completes_through_the_c_surface(api, tmp_path):
    out = tmp_path / "dolb_capi_run"
    steps, mlups = api.run({"case.kind": "tgv", "case.L": "8", "case.Re": "8", "case.Ma": "0.1",
                            "run.tmax": "10", "run.output_every": "5", "run.out": str(out)})
    assert steps == 10 and mlups > 0.0
    assert (out / "series.csv").exists()


def _sha(path):
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(RUNNER_CASES))
def test_run_artefacts_match_reference(api, name, tmp_path):
    """series.csv, profiles.csv, manifest and DOLB1 dumps byte-identical to the
    reference's dolb_run on the same configuration."""
    with open(os.path.join(GOLD, "index.json")) as fh:
        want = json.load(fh)[name]
    out = str(tmp_path / "out")
    steps, mlups = api.run(resolve_paths(RUNNER_CASES[name], out))
    assert steps == want["steps"] and mlups > 0
    for f in ("series.csv", "profiles.csv"):
        g = os.path.join(GOLD, name, f)
        assert os.path.exists(g) == os.path.exists(os.path.join(out, f)), f
        if os.path.exists(g):
            with open(g) as a, open(os.path.join(out, f)) as b:
                assert b.read() == a.read(), f
    with open(os.path.join(GOLD, name, "manifest")) as a, open(os.path.join(out, "manifest")) as b:
        assert normalize_manifest(b.read(), out) == a.read()
    for dump, sha in want["dumps"].items():
        assert _sha(os.path.join(out, dump)) == sha, dump
    with open(os.path.join(out, "perf.csv")) as fh:
        head, row = fh.read().splitlines()[:2]
    cols = row.split(",")
    assert head == want["perf_header"]
    assert cols[0] == want["perf_fixed"]["cells"] and cols[1] == want["perf_fixed"]["steps"]
    # device name, bytes per cell, peak: identical; fraction columns depend on the measured MLUPS
    assert cols[4:7] == want["perf_fixed"]["tail"][:3]


@pytest.mark.gpu
def test_manifest_replay_reproduces_series(api, tmp_path):
    first = str(tmp_path / "a")
    api.run(resolve_paths(RUNNER_CASES["cavity16_trt_f32"], first))
    with api.config() as cfg:
        cfg.load(os.path.join(first, "manifest"))
        second = str(tmp_path / "b")
        cfg.set("run.out", second)
        cfg.run()
    with open(os.path.join(first, "series.csv")) as a, open(os.path.join(second, "series.csv")) as b:
        assert a.read() == b.read()


@pytest.mark.gpu
def test_dispatch_set_missing_a_used_chain_fails(api, tmp_path):
    values = {"case.kind": "cavity", "case.L": "16", "run.tmax": "4", "run.output_every": "2",
              "dispatch.models": "COLL_BGK", "run.out": str(tmp_path)}
    with pytest.raises(DolbError) as e:
        api.run(values)
    assert e.value.status == DISPATCH
    assert "BounceBack" in e.value.message and "not part of the dispatch set" in e.value.message
    with pytest.raises(DolbError) as e:
        api.run(dict(values, **{"dispatch.models": "COLL_BGK,NoSuchModel"}))
    assert e.value.status == CONFIG


@pytest.mark.gpu
def test_fast_arith_and_device_keys(api, tmp_path):
    out = str(tmp_path / "f")
    steps, _ = api.run(dict(resolve_paths(RUNNER_CASES["tgv16_bgk_f64"], out), **{"run.arith": "fast",
                                                                                 "run.devices": "0"}))
    assert steps == 40
    with open(os.path.join(out, "manifest")) as fh:
        text = fh.read()
    assert "arith = fast" in text and "devices = 0" in text
    shutil.rmtree(out)


@pytest.mark.gpu
@pytest.mark.parametrize("name,extra,dumps", [
    ("sphere48_trt_f64", {"run.porous": "masked"}, False),   # NoDynamics segments skipped
    ("sphere48_trt_f64", {"run.porous": "lists"}, False),
    ("tgv16_bgk_f64", {"run.layout": "aa"}, True),             # in-place AA streaming
    ("cavity16_trt_f32", {"run.layout": "aa"}, False),
    ("tgv16_blocks_f64", {"run.layout": "aa"}, False),         # AA on 3 linked z-slabs
    ("c1_cavity64_bgk_f64", {"run.layout": "aa"}, True),       # config 1, 8 AA z-slabs
])
def test_device_variants_keep_the_reference_series(api, name, extra, dumps, tmp_path):
    """Device-runtime variants behind run.porous / run.layout: series.csv (and,
    where every cell is updated, the DOLB1 dumps) stay byte-identical to the
    reference's dolb_run -- the masked / sparse porous sweeps only leave
    never-consumed solid-cell values stale, which the diagnostics never read."""
    with open(os.path.join(GOLD, "index.json")) as fh:
        want = json.load(fh)[name]
    out = str(tmp_path / "v")
    steps, _ = api.run(dict(resolve_paths(RUNNER_CASES[name], out), **extra))
    assert steps == want["steps"]
    with open(os.path.join(GOLD, name, "series.csv")) as a, open(os.path.join(out, "series.csv")) as b:
        assert b.read() == a.read()
    if dumps:
        for dump, sha in want["dumps"].items():
            assert _sha(os.path.join(out, dump)) == sha, dump
    with open(os.path.join(out, "manifest")) as fh:
        text = fh.read()
    for k, v in extra.items():
        assert f"{k.split('.')[1]} = {v}" in text


def test_variant_keys_validated(api, tmp_path):
    for key, bad, msg in (("run.layout", "soa", 'unknown layout "soa"'),
                          ("run.porous", "holes", 'unknown porous sweep "holes"'),
                          ("run.arith", "approx", 'unknown arithmetic mode "approx"')):
        with pytest.raises(DolbError) as e:
            api.run({key: bad, "run.out": str(tmp_path)})
        assert e.value.status == CONFIG and msg in e.value.message


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [64, 32])
def test_d3q27_through_dolb_run(api, oracle, bits, tmp_path):
    """Config 2's lattice through the public API (case.lattice = d3q27, a
    device-runtime extension: the reference is D3Q19 only): the DOLB1 dump of
    a TGV RR run equals the oracle's D3Q27 restatement bit for bit."""
    import numpy as np
    from paper_2506_09242_b200.dolb import read_field_dump
    from pyoracle import RR, Case
    out = str(tmp_path / "q27")
    steps, _ = api.run({"case.kind": "tgv", "case.L": "16", "case.Re": "400", "case.Ma": "0.1",
                        "case.collision": "rr", "case.lattice": "d3q27", "case.precision": f"f{bits}",
                        "run.tmax": "20", "run.output_every": "10", "run.dump_every": "20", "run.out": out})
    assert steps == 20
    dims, prec, got = read_field_dump(os.path.join(out, "dump_00000020.dolb"))
    assert dims == (16, 16, 16) and prec == bits // 8
    dt = np.float64 if bits == 64 else np.float32
    want = oracle.run_case(Case(kind="tgv", L=16, Re=400.0, Ma=0.1, collision=RR, q=27), dt, 20)
    assert np.array_equal(got, np.asarray(want, np.float64).reshape(-1))
    with open(os.path.join(out, "manifest")) as fh:
        assert "lattice = d3q27" in fh.read()


def test_d3q27_porous_rejected(api, tmp_path):
    with pytest.raises(DolbError) as e:
        api.run({"case.kind": "porous", "case.geometry": "plates", "case.lattice": "d3q27",
                 "run.out": str(tmp_path)})
    assert e.value.status == CONFIG and "d3q27" in e.value.message
