"""Full-size parity checksums that need the GPU box's host (197 GiB RAM, 16+ cores).

TEST INFRASTRUCTURE ONLY. Run ON THE GPU BOX (the build container has 62 GB):

    python tests/golden/make_golden_box.py [--out gpurun_out/golden_box.json] [name ...]

and copy the entries into tests/golden/golden_full.json. Every entry records
the dlb_lattice_checksum definition (per direction: sum of
bits(double(f_i) + 0.0) * (global cell index + 1) mod 2^64) of the state
after `steps` steps:

  c5  Taylor-Green D3Q19 BGK fp32 at 896^3 (1024^3 needs ~187 GB in the
      reference's block layout; 896^3 is the largest multiple of 128 that
      leaves headroom): the UNMODIFIED reference (oracle/_ref,
      MultiBlockRun<float>, 16 workers x z-blocks), checksum streamed over its
      blocks (no gather copy).
  c4  the bench geometry itself: seeded sphere pack 600^3 (R = 8, porosity
      0.20, mt19937_64 seed 20250611, written by the product's input generator
      in the reference's raw voxel format and loaded by the reference's
      load_voxels) + 40/40 buffers = 680 x 600 x 600, TRT fp64, velocity
      drive: the reference, checksum of every cell and of the cells whose
      chain is not NoDynamics (what the masked sweep must match).
  c2  Taylor-Green Re = 1600 D3Q27 RR fp64 256^3, 100 steps: the CPU oracle
      restatement (oracle/lbm_oracle.c, all host threads). D3Q27 has no
      reference implementation: parity unpinned.
"""
import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from pyoracle import BGK, RR, TRT, Case, Oracle, Reference, canonical_checksum  # noqa: E402

BOX_CASES = {
    "tgv896_bgk_f32_c5_box": dict(kind="tgv", L=896, Re=1600.0, Ma=0.2, collision=BGK, bits=32, steps=20,
                                  workers=16, impl="reference"),
    "porous680x600x600_trt_f64_c4_box": dict(kind="porous", L=600, Ma=0.01, collision=TRT, bits=64, steps=10,
                                             tau=1.0, upstream=40, downstream=40, sphere=dict(
                                                 n=600, radius=8.0, porosity=0.20, seed=20250611),
                                             workers=16, impl="reference"),
    "tgv256_rr27_f64_c2_box": dict(kind="tgv", L=256, Re=1600.0, Ma=0.2, collision=RR, q=27, bits=64, steps=100,
                                   impl="oracle"),
}


def sphere_raw(sp):
    """The c4 geometry through the product's generator (dlb_case_sphere_pack),
    as the reference's raw voxel file; returns (path, porosity, sha256)."""
    import paper_2506_09242_b200 as dlb
    n = sp["n"]
    vox, phi = dlb.sphere_pack((n, n, n), radius=sp["radius"], porosity=sp["porosity"], seed=sp["seed"])
    path = os.path.join(tempfile.gettempdir(), f"dlb_sphere_{n}_{sp['seed']}.raw")
    vox.tofile(path)
    return path, float(phi), hashlib.sha256(vox.tobytes()).hexdigest()


def make(spec):
    s = {k: v for k, v in spec.items() if k not in ("bits", "steps", "workers", "impl", "sphere")}
    extra = {}
    if "sphere" in spec:
        path, phi, sha = sphere_raw(spec["sphere"])
        n = spec["sphere"]["n"]
        s.update(geometry=path, voxel_dims=(n, n, n))
        extra = {"porosity": phi, "voxels_sha256": sha}
    return Case(**s), extra


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    out_path = os.path.join(ROOT, "gpurun_out", "golden_box.json")
    if "--out" in sys.argv:
        out_path = sys.argv[sys.argv.index("--out") + 1]
        args = [a for a in args if a != out_path]
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    print(f"host: {os.cpu_count()} cpus, "
          f"{os.sysconf('SC_PAGE_SIZE') * os.sysconf('SC_PHYS_PAGES') / 2**30:.0f} GiB", flush=True)
    for name, spec in BOX_CASES.items():
        if (args and name not in args) or name in out:
            continue
        t = time.time()
        case, extra = make(spec)
        entry = {"spec": {k: v for k, v in spec.items()}, **extra}
        if spec["impl"] == "reference":
            w = spec.get("workers", 16)
            cs, act = Reference().checksum_masked(case, spec["bits"], spec["steps"], grid=(1, 1, w), workers=w)
            entry["checksum"] = [str(v) for v in cs]
            entry["checksum_active"] = [str(v) for v in act]
        else:
            dt = np.float64 if spec["bits"] == 64 else np.float32
            pops = Oracle().run_case(case, dt, spec["steps"], nthreads=os.cpu_count())
            entry["checksum"] = [str(v) for v in canonical_checksum(pops, q=case.q)]
            del pops
        entry["seconds"] = round(time.time() - t, 1)
        out[name] = entry
        print(f"{name}: {entry['seconds']} s", flush=True)
        with open(out_path, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
