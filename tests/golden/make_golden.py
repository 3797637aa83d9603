"""Generate tests/golden/golden.json from the UNMODIFIED reference solver.

Run in the build container (needs oracle/_ref/libdolb_refshim.so, built from
/root/reference/proj by `make -C oracle ref`):

    python tests/golden/make_golden.py          # golden.json
    python tests/golden/make_golden.py --full   # golden_full.json (full-size checksums)
    python tests/golden/make_golden.py --diag   # golden_diag.json (sampling step)

Each entry records the reference's gather_populations() after `steps` steps
(MultiBlockRun<T>, 8 workers x z-blocks — decomposition does not change the
bits, test_multiblock.cpp:234-256) as a sha256 of the float64 values with -0
folded to +0, plus summary values. Porous entries read sphere48.raw, a mask
written by the product's seeded sphere-pack generator in the reference's raw
voxel format (committed next to this file).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)
from pyoracle import Reference, canonical_checksum, canonical_hash  # noqa: E402
from golden_cases import CASES, DIAG_CASES, FULL_CASES, make_case  # noqa: E402


def full():
    """Full-size configs: only the order-independent checksum is recorded
    (dlb_lattice_checksum definition), the state is too large to hash in Python."""
    ref = Reference()
    path = os.path.join(HERE, "golden_full.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name, spec in FULL_CASES.items():
        if name in out:
            continue
        case = make_case(spec)
        t = time.time()
        cs = ref.checksum(case, spec["bits"], spec["steps"], grid=(1, 1, spec.get("workers", 8)),
                          workers=spec.get("workers", 8))
        out[name] = {"spec": spec, "checksum": [str(v) for v in cs]}
        print(f"{name}: {time.time() - t:.1f}s", flush=True)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)


def diag():
    """Sampling-step values (kinetic energy, enstrophy, cavity convergence sums,
    porous permeability extras) of the reference's runner arithmetic on its own
    gathered fields, stored as exact float hex strings."""
    ref = Reference()
    out = {}
    for name, (a, b) in DIAG_CASES.items():
        spec = CASES[name]
        t = time.time()
        vals = ref.sample(make_case(spec), spec["bits"], a, b)
        out[name] = {"steps": [a, b], "values": {k: float(v).hex() for k, v in vals.items()}}
        print(f"{name}: {time.time() - t:.1f}s k={vals['k']:.6g} eps={vals['eps']:.6g}", flush=True)
    with open(os.path.join(HERE, "golden_diag.json"), "w") as f:
        json.dump(out, f, indent=1)


def main():
    if "--full" in sys.argv:
        return full()
    if "--diag" in sys.argv:
        return diag()
    ref = Reference()
    out = {}
    for name, spec in CASES.items():
        case = make_case(spec)
        t = time.time()
        pops = ref.run_case(case, spec["bits"], spec["steps"], grid=(1, 1, spec.get("workers", 4)),
                            workers=spec.get("workers", 4))
        dt = time.time() - t
        q = 19
        n = pops.size // q
        idx = np.linspace(0, pops.size - 1, 16).astype(np.int64)
        out[name] = {
            "spec": spec,
            "sha256": canonical_hash(pops),
            "sum": float(pops.sum()),
            "absmax": float(np.abs(pops).max()),
            "mass": float(pops.reshape(q, n).sum()),
            "sample_index": idx.tolist(),
            "sample": [float(v) for v in pops[idx]],
        }
        print(f"{name}: {dt:.1f}s sha={out[name]['sha256'][:16]}", flush=True)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
