"""Public-API throughput: the reference's dolb_run entry point (include/dolb.h)
on full-size configurations, MLUPS as the reference's runner reports it
(advance time only, runner.cpp:703-709), plus the wall time of the call."""
import json
import sys
import tempfile
import time

sys.path.insert(0, ".")
from paper_2506_09242_b200.runner import Dolb  # noqa: E402

CASES = {
    "c5 TGV 1024^3 BGK f32": {"case.kind": "tgv", "case.L": "1024", "case.precision": "f32",
                               "run.tmax": "200", "run.output_every": "100"},
    "c3 cavity 512^3 TRT f32": {"case.kind": "cavity", "case.L": "512", "case.collision": "trt",
                                "case.precision": "f32", "run.tmax": "400", "run.output_every": "200"},
    "c1 cavity 64^3 BGK f64": {"case.kind": "cavity", "case.L": "64", "run.tmax": "1000",
                               "run.output_every": "250"},
}
api = Dolb()
for name, cfg in CASES.items():
    with tempfile.TemporaryDirectory() as out:
        t = time.perf_counter()
        steps, mlups = api.run(dict(cfg, **{"run.out": out}))
        wall = time.perf_counter() - t
        print(json.dumps({"case": name, "steps": steps, "mlups_reported": mlups, "wall_s": wall,
                          "series": open(out + "/series.csv").read().splitlines()[-1]}), flush=True)
