"""Full-size parity of the BASELINE configurations (GPU).

The expected values are the dlb_lattice_checksum of the reference's state
(or, for D3Q27, the CPU oracle's) at the configured sizes, generated on the
GPU box's host (197 GiB RAM) by tests/golden/make_golden_box.py and committed
in tests/golden/golden_full.json:

  c5  TGV D3Q19 BGK fp32 at 896^3, 20 steps: the unmodified reference
      (oracle/_ref MultiBlockRun<float>, 16 workers). 1024^3 does not fit the
      reference's block layout in host RAM (~187 GB); the 1024^3 run itself is
      checked for layout / decomposition invariance in test_gpu_parity.py.
  c4  the bench geometry: sphere pack 600^3 (R 8, porosity 0.20, seed
      20250611) + 40/40 buffers = 680 x 600 x 600, TRT fp64, 10 steps: the
      reference; dense sweep = every cell, masked sweep = every non-NoDynamics
      cell.
  c2  TGV D3Q27 RR fp64 256^3, 100 steps: the oracle (no D3Q27 reference
      exists: parity unpinned).

Bit-identical (exact arithmetic) is the bar for all of them.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2506_09242_b200 as dlb

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_full.json")))
LT = {0: dlb.LinkType.BGK, 1: dlb.LinkType.TRT, 2: dlb.LinkType.RR}


def setup_of(spec):
    q = spec.get("q", 19)
    if spec["kind"] == "porous":
        sp = spec["sphere"]
        n = sp["n"]
        vox, phi = dlb.sphere_pack((n, n, n), radius=sp["radius"], porosity=sp["porosity"], seed=sp["seed"])
        cfg = dlb.CaseConfig(kind="porous", L=spec["L"], Ma=spec["Ma"], collision=LT[spec["collision"]], q=q,
                             tau=spec["tau"], upstream=spec["upstream"], downstream=spec["downstream"])
        return dlb.init_porous(cfg, solid=(vox == 255)), hashlib.sha256(vox.tobytes()).hexdigest(), phi
    cfg = dlb.CaseConfig(kind=spec["kind"], L=spec["L"], Re=spec["Re"], Ma=spec["Ma"],
                         collision=LT[spec["collision"]], q=q)
    return (dlb.init_tgv(cfg) if spec["kind"] == "tgv" else dlb.init_cavity(cfg)), None, None


def expect(name, key="checksum"):
    return [int(v) for v in GOLD[name][key]]


@pytest.mark.parametrize("layout,slabs", [("twopop", 1), ("aa", 1), ("twopop", 4), ("aa", 4)])
def test_config5_896_matches_reference(layout, slabs):
    name = "tgv896_bgk_f32_c5_box"
    spec = GOLD[name]["spec"]
    setup, _, _ = setup_of(spec)
    run = dlb.build_run(setup, precision=32, layout=layout, slabs=slabs)
    run.advance(spec["steps"])
    assert run.checksum() == expect(name)


@pytest.mark.parametrize("variant", ["dense", "masked", "compact"])
def test_config4_bench_geometry_matches_reference(variant, monkeypatch):
    name = "porous680x600x600_trt_f64_c4_box"
    g = GOLD[name]
    spec = g["spec"]
    setup, sha, phi = setup_of(spec)
    # the geometry is the one the reference loaded (same generator, same bytes)
    assert sha == g["voxels_sha256"] and phi == g["porosity"]
    if variant == "compact":
        monkeypatch.setenv("DLB_POROUS_COMPACT", "1")
    run = dlb.build_run(setup, precision=64, skip_nodynamics=variant != "dense")
    del setup
    if variant == "compact":
        assert "k_cmp" in run.kernel_name()
    run.advance(spec["steps"])
    if variant == "dense":
        assert run.checksum() == expect(name)
    else:
        assert run.checksum(active_only=True) == expect(name, "checksum_active")


@pytest.mark.parametrize("slabs", [1, 2])
def test_config2_256_matches_oracle(slabs):
    name = "tgv256_rr27_f64_c2_box"
    spec = GOLD[name]["spec"]
    setup, _, _ = setup_of(spec)
    run = dlb.build_run(setup, precision=64, slabs=slabs)
    run.advance(spec["steps"])
    assert run.checksum() == expect(name)
