"""GPU-side checksums of the full-size parity configurations (tools probe; the
committed tests are tests/test_full_parity.py). Prints one JSON object per
case (and writes gpurun_out/gpu_full.json) with the dlb_lattice_checksum of the
state after the steps tests/golden/make_golden_box.py runs on the reference /
oracle.

    python tools/full_parity_gpu.py [name ...]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402

import paper_2506_09242_b200 as dlb  # noqa: E402
from make_golden_box import BOX_CASES  # noqa: E402


def gpu_checksums(name, spec, variant):
    lt = {0: dlb.LinkType.BGK, 1: dlb.LinkType.TRT, 2: dlb.LinkType.RR}[spec["collision"]]
    q = spec.get("q", 19)
    kw = {}
    if spec["kind"] == "porous":
        sp = spec["sphere"]
        n = sp["n"]
        vox, _ = dlb.sphere_pack((n, n, n), radius=sp["radius"], porosity=sp["porosity"], seed=sp["seed"])
        cfg = dlb.CaseConfig(kind="porous", L=spec["L"], Ma=spec["Ma"], collision=lt, q=q, tau=spec["tau"],
                             upstream=spec["upstream"], downstream=spec["downstream"])
        setup = dlb.init_porous(cfg, solid=(vox == 255))
        del vox
        kw["skip_nodynamics"] = variant == "masked"
    else:
        cfg = dlb.CaseConfig(kind=spec["kind"], L=spec["L"], Re=spec["Re"], Ma=spec["Ma"], collision=lt, q=q)
        setup = dlb.init_tgv(cfg) if spec["kind"] == "tgv" else dlb.init_cavity(cfg)
        if variant == "aa":
            kw["layout"] = "aa"
    run = dlb.build_run(setup, precision=spec["bits"], **kw)
    run.advance(spec["steps"])
    run.synchronize()
    cs = run.checksum()
    out = {"checksum": [str(v) for v in cs], "kernel": run.kernel_name()}
    if kw.get("skip_nodynamics"):
        out["checksum_active"] = [str(v) for v in run.checksum(active_only=True)]
    return out


def main():
    names = sys.argv[1:] or list(BOX_CASES)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "gpu_full.json")
    res = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        spec = BOX_CASES[name]
        variants = {"porous": ["dense", "masked"], "tgv": ["twopop", "aa"]}.get(spec["kind"], ["twopop"])
        if spec.get("q", 19) == 27:
            variants = ["twopop"]
        for v in variants:
            t = time.time()
            r = gpu_checksums(name, spec, v)
            r["seconds"] = round(time.time() - t, 1)
            res[f"{name}:{v}"] = r
            print(json.dumps({f"{name}:{v}": r}), flush=True)
            with open(path, "w") as f:
                json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
