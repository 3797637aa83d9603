"""Runner configurations whose artefacts are pinned against the reference's
dolb_run (tests/golden/runner/, made by make_runner_golden.py). Small enough
for the reference's single-worker CPU path to finish in seconds."""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SPHERE = os.path.join(HERE, "sphere48.raw")

RUNNER_CASES = {
    "tgv16_bgk_f64": {"case.kind": "tgv", "case.L": "16", "case.Re": "100", "case.Ma": "0.1",
                      "run.tmax": "40", "run.output_every": "10", "run.dump_every": "20"},
    "tgv16_rr_f32": {"case.kind": "tgv", "case.L": "16", "case.Re": "400", "case.Ma": "0.1",
                     "case.collision": "rr", "case.precision": "f32", "run.tmax": "30",
                     "run.output_every": "10", "run.dump_every": "30"},
    "tgv12_les_trt_f64": {"case.kind": "tgv", "case.L": "12", "case.Re": "1600", "case.Ma": "0.1",
                          "case.collision": "trt", "case.smagorinsky": "0.14", "run.tmax": "1tc",
                          "run.output_every": "8"},
    "tgv16_blocks_f64": {"case.kind": "tgv", "case.L": "16", "case.Re": "100", "case.Ma": "0.1",
                         "run.tmax": "20", "run.output_every": "10", "run.blocks": "1,1,3",
                         "run.workers": "3"},
    "cavity16_trt_f32": {"case.kind": "cavity", "case.L": "16", "case.Re": "100", "case.Ma": "0.1",
                         "case.collision": "trt", "case.precision": "f32", "run.tmax": "60",
                         "run.output_every": "20", "run.avg_from": "0"},
    "cavity20_bgk_f64": {"case.kind": "cavity", "case.L": "20", "case.Re": "200", "case.Ma": "0.1",
                         "run.tmax": "2tc", "run.output_every": "100", "run.blocks": "1,1,2",
                         "run.perf_device": "A100-SXM4-40GB"},
    "plates20_trt_vel_f64": {"case.kind": "porous", "case.geometry": "plates", "case.L": "20",
                             "case.H": "6", "case.upstream": "4", "case.downstream": "4",
                             "run.tmax": "400", "run.output_every": "100"},
    "plates20_rr_pres_f32": {"case.kind": "porous", "case.geometry": "plates", "case.L": "20",
                             "case.H": "6", "case.upstream": "4", "case.downstream": "4",
                             "case.collision": "rr", "case.drive": "pressure", "case.tau": "0.9",
                             "case.precision": "f32", "run.tmax": "300", "run.output_every": "100"},
    "plates16_steady_f64": {"case.kind": "porous", "case.geometry": "plates", "case.L": "16",
                            "case.H": "4", "case.upstream": "4", "case.downstream": "4",
                            "run.tmax": "steady", "run.steady_tol": "1e-4", "run.max_steps": "3000",
                            "run.output_every": "50"},
    # config 1 through the public API: lid-driven cavity 64^3 D3Q19 BGK fp64, 1000 steps
    "c1_cavity64_bgk_f64": {"case.kind": "cavity", "case.L": "64", "case.Re": "1000", "case.Ma": "0.1",
                            "run.tmax": "1000", "run.output_every": "250", "run.blocks": "1,1,8",
                            "run.workers": "8", "run.dump_every": "1000"},
    # config 3 shape at reduced size: cavity TRT fp32
    "c3_cavity96_trt_f32": {"case.kind": "cavity", "case.L": "96", "case.Re": "1000", "case.Ma": "0.1",
                            "case.collision": "trt", "case.precision": "f32", "run.tmax": "200",
                            "run.output_every": "100", "run.blocks": "1,1,8", "run.workers": "8",
                            "run.avg_from": "0"},
    "sphere48_trt_f64": {"case.kind": "porous", "case.geometry": "@SPHERE", "case.voxel_dims": "48,48,48",
                         "case.upstream": "8", "case.downstream": "8", "run.tmax": "200",
                         "run.output_every": "50", "run.dump_every": "200"},
}


def resolve_paths(cfg: dict, out_dir: str) -> dict:
    v = {k: (SPHERE if val == "@SPHERE" else val) for k, val in cfg.items()}
    v["run.out"] = out_dir
    return v


def normalize_manifest(text: str, out_dir: str) -> str:
    return text.replace(out_dir, "@OUT").replace(SPHERE, "@SPHERE")
