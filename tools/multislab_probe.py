"""Single-process multi-slab stepping cost (dlb_lattices_step): config 1's
64^3 cavity (and a 256^3 TGV) as 1, 2, 4, 8 linked slabs on one GPU, wall
clock per step over many steps (host enqueue vs device time).

    python tools/multislab_probe.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09242_b200 as dlb  # noqa: E402

for kind, L, bits, n in (("cavity", 64, 64, 1000), ("tgv", 256, 32, 200)):
    for slabs in (1, 2, 4, 8):
        cfg = dlb.CaseConfig(kind=kind, L=L, Re=1000.0, Ma=0.1)
        setup = dlb.init_cavity(cfg) if kind == "cavity" else dlb.init_tgv(cfg)
        run = dlb.build_run(setup, precision=bits, slabs=slabs)
        run.advance(10)
        run.synchronize()
        t0 = time.perf_counter()
        run.advance(n)
        t1 = time.perf_counter()
        run.synchronize()
        t2 = time.perf_counter()
        print(json.dumps({"case": f"{kind}{L} fp{bits}", "slabs": slabs, "steps": n,
                          "us_per_step": round((t2 - t0) / n * 1e6, 2),
                          "host_enqueue_us_per_step": round((t1 - t0) / n * 1e6, 2),
                          "mlups": round(L ** 3 * n / (t2 - t0) / 1e6)}), flush=True)
        del run
