"""Golden case specifications shared by make_golden.py and the tests."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle"))
from pyoracle import BGK, RR, TRT, Case  # noqa: E402

SPHERE_RAW = os.path.join(HERE, "sphere48.raw")
SPHERE_DIMS = (48, 48, 48)

# name -> case spec. bits = storage precision; steps = reference steps.
CASES = {
    # test_accelerated.cpp:131-168 (golden dump TGV16, 10 steps)
    "tgv16_bgk_f64": dict(kind="tgv", L=16, Re=8.0, Ma=0.1, collision=BGK, bits=64, steps=10),
    # test_accelerated.cpp:302-328 (float path, TGV12, 5 steps)
    "tgv12_bgk_f32": dict(kind="tgv", L=12, Re=8.0, Ma=0.1, collision=BGK, bits=32, steps=5),
    # config 1 at full size: lid-driven cavity D3Q19 BGK 64^3 fp64, 1000 steps
    "cavity64_bgk_f64_c1": dict(kind="cavity", L=64, Re=1000.0, Ma=0.1, collision=BGK, bits=64,
                                steps=1000, workers=8),
    "cavity32_trt_f32": dict(kind="cavity", L=32, Re=1000.0, Ma=0.1, collision=TRT, bits=32, steps=200),
    "cavity24_rr_f64": dict(kind="cavity", L=24, Re=400.0, Ma=0.1, collision=RR, bits=64, steps=100),
    "tgv32_trt_f64": dict(kind="tgv", L=32, Re=400.0, Ma=0.1, collision=TRT, bits=64, steps=50),
    "tgv32_rr_f64": dict(kind="tgv", L=32, Re=1600.0, Ma=0.2, collision=RR, bits=64, steps=50),
    "tgv32_rr_f32": dict(kind="tgv", L=32, Re=1600.0, Ma=0.2, collision=RR, bits=32, steps=50),
    "tgv24_smag_bgk_f64": dict(kind="tgv", L=24, Re=1600.0, Ma=0.2, collision=BGK, bits=64, steps=40,
                               smagorinsky_c=0.16),
    "tgv24_smag_trt_f32": dict(kind="tgv", L=24, Re=1600.0, Ma=0.2, collision=TRT, bits=32, steps=40,
                               smagorinsky_c=0.16),
    # config 5 reduced (128^3, <= 3 t_c)
    "tgv128_bgk_f32_c5": dict(kind="tgv", L=128, Re=1600.0, Ma=0.2, collision=BGK, bits=32, steps=100,
                              workers=8),
    # config 3 reduced (cavity TRT fp32)
    "cavity128_trt_f32_c3": dict(kind="cavity", L=128, Re=1000.0, Ma=0.1, collision=TRT, bits=32,
                                 steps=20, workers=8),
    # porous plates with regularized velocity / pressure drives
    "plates16_trt_vel_f64": dict(kind="porous", L=16, Ma=0.01, collision=TRT, bits=64, steps=200,
                                 plate_layers=6, upstream=4, downstream=4, tau=1.0),
    "plates16_trt_pres_f32": dict(kind="porous", L=16, Ma=0.01, collision=TRT, bits=32, steps=200,
                                  plate_layers=6, upstream=4, downstream=4, tau=0.8, drive="pressure"),
    "plates16_rr_vel_f64": dict(kind="porous", L=16, Ma=0.01, collision=RR, bits=64, steps=100,
                                plate_layers=6, upstream=4, downstream=4, tau=0.9),
    "plates16_bgk_pres_f64": dict(kind="porous", L=16, Ma=0.01, collision=BGK, bits=64, steps=100,
                                  plate_layers=6, upstream=4, downstream=4, tau=1.0, drive="pressure"),
    # config 4 reduced: seeded sphere pack (~20% porosity) + 8/8 buffers, TRT fp64
    "sphere48_trt_f64_c4": dict(kind="porous", L=48, Ma=0.01, collision=TRT, bits=64, steps=200,
                                geometry="sphere48", voxel_dims=SPHERE_DIMS, upstream=8,
                                downstream=8, tau=1.0, workers=8),
}


def make_case(spec) -> Case:
    s = dict(spec)
    for k in ("bits", "steps", "workers"):
        s.pop(k, None)
    if s.get("geometry") == "sphere48":
        s["geometry"] = SPHERE_RAW
    return Case(**s)


# Full-size BASELINE configs the reference can run in the build container
# (62 GB RAM): checksums only (tests/golden/golden_full.json).
FULL_CASES = {
    # config 3 per-GPU size: lid-driven cavity D3Q19 TRT 512^3 fp32
    "cavity512_trt_f32_c3_full": dict(kind="cavity", L=512, Re=1000.0, Ma=0.1, collision=TRT, bits=32,
                                      steps=6, workers=8),
    # config 1 (also hashed in golden.json)
    "cavity64_bgk_f64_c1_full": dict(kind="cavity", L=64, Re=1000.0, Ma=0.1, collision=BGK, bits=64,
                                     steps=1000, workers=8),
}

# Sampling-step goldens (runner.cpp:346-448 on the reference's own fields):
# case name -> (steps before the velocity snapshot, steps after it).
DIAG_CASES = {
    "tgv16_bgk_f64": (5, 5),
    "tgv12_bgk_f32": (3, 2),
    "tgv32_rr_f64": (25, 25),
    "tgv24_smag_trt_f32": (20, 20),
    "tgv128_bgk_f32_c5": (50, 50),
    "cavity64_bgk_f64_c1": (500, 500),
    "cavity32_trt_f32": (100, 100),
    "cavity24_rr_f64": (50, 50),
    "plates16_trt_vel_f64": (100, 100),
    "plates16_trt_pres_f32": (100, 100),
    "sphere48_trt_f64_c4": (100, 100),
}
