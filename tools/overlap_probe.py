"""Halo / interior overlap of linked z-slabs on ONE GPU.

1. Step time of the same L^3 TGV D3Q19 BGK fp32 lattice as 1, 2, 4, 8 linked
   slabs in one process (wall clock over `n` steps after warm-up, device
   synchronised on both sides): the protocol cost (halo wait, boundary /
   interior split, peer pushes, system-scope fences) on top of the single
   slab, which runs with in-kernel periodic wrap and no exchange.
2. With DLB_TRACE_HALO=1 (graphs off): per-step timeline of slab 0 of a
   2-slab run -- halo wait and boundary launch on the high-priority halo
   stream against the interior launch on the main stream.

    python tools/overlap_probe.py [L] [--trace | --self] [--aa]

--aa: the same measurements on AA in-place slabs (one population array).

3. --self: one slab linked to itself (z wrap through its own halo protocol),
   serialised (DLB_HALO_OVERLAP=0) vs overlapped, against the unlinked slab:
   the single-GPU proxy of one slab per GPU.
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09242_b200 as dlb  # noqa: E402
from paper_2506_09242_b200 import _capi  # noqa: E402

L = int(next((a for a in sys.argv[1:] if a.isdigit()), 512))
n = 40
LAYOUT = "aa" if "--aa" in sys.argv else "twopop"


def step_time(slabs):
    cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
    run = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=slabs, layout=LAYOUT)
    run.advance(6)
    run.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        run.advance(n)
        run.synchronize()
        best = min(best, (time.perf_counter() - t) / n)
    del run
    return best


def self_linked_time(link, overlap):
    """One slab, z-periodic through its own halo protocol (linked to itself):
    the per-GPU step of a z-slab run (wait, boundary + push, interior) on one
    GPU, vs the same lattice with in-kernel wrap."""
    os.environ["DLB_HALO_OVERLAP"] = "1" if overlap else "0"
    cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
    run = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=1, layout=LAYOUT)
    h = run.slabs[0].handle
    if link:
        _capi.check(_capi.lib().dlb_lattice_link_local(h, h))
        if LAYOUT == "aa":  # linking clears an AA slab's state: refill
            run.fill_tgv(L, 0.2 / 3 ** 0.5)
        _capi.check(_capi.lib().dlb_lattice_exchange(h))
    run.advance(6)
    run.synchronize()
    best = min(run.time_steps(n) / n for _ in range(3))
    cs = run.checksum()
    del run
    return best, cs


def trace(slabs=2, steps=6, self_link=False):
    cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
    run = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=slabs, layout=LAYOUT)
    if self_link:
        h0 = run.slabs[0].handle
        _capi.check(_capi.lib().dlb_lattice_link_local(h0, h0))
        if LAYOUT == "aa":
            run.fill_tgv(L, 0.2 / 3 ** 0.5)
        _capi.check(_capi.lib().dlb_lattice_exchange(h0))
    run.advance(2)
    run.synchronize()
    h = run.slabs[0].handle
    nn = C.c_size_t()
    _capi.check(_capi.lib().dlb_lattice_halo_trace(h, None, 0, C.byref(nn)))  # drop warm-up events
    run.advance(steps)
    run.synchronize()
    _capi.check(_capi.lib().dlb_lattice_halo_trace(h, None, 0, C.byref(nn)))
    buf = (C.c_double * nn.value)()
    _capi.check(_capi.lib().dlb_lattice_halo_trace(h, buf, nn.value, C.byref(nn)))
    t = list(buf)
    rows = []
    for k in range(len(t) // 5):
        w0, w1, b1, i0, i1 = t[5 * k:5 * k + 5]
        rows.append({"step": k, "wait_ms": [round(w0, 4), round(w1, 4)], "boundary_end_ms": round(b1, 4),
                     "interior_ms": [round(i0, 4), round(i1, 4)],
                     "halo_branch_inside_interior": bool(i0 <= w0 + 1e-3 and b1 <= i1)})
    return rows


if "--self" in sys.argv and "--trace" not in sys.argv:
    ref = None
    for link, overlap in ((False, True), (True, False), (True, True)):
        ms, cs = self_linked_time(link, overlap)
        ref = ref or ms
        same = None
        print(json.dumps({"L": L, "layout": LAYOUT, "self_linked": link, "overlap": overlap if link else None,
                          "ms_per_step": round(ms, 4), "mlups": round(L ** 3 / ms / 1e3),
                          "vs_unlinked": round(ms / ref, 4), "checksum0": str(cs[0])}), flush=True)
elif "--trace" in sys.argv:
    os.environ["DLB_TRACE_HALO"] = "1"
    for r in (trace(slabs=1, self_link=True) if "--self" in sys.argv else trace()):
        print(json.dumps(r), flush=True)
else:
    base = None
    for slabs in (1, 2, 4, 8):
        dt = step_time(slabs)
        base = base or dt
        print(json.dumps({"L": L, "layout": LAYOUT, "slabs": slabs, "ms_per_step": round(dt * 1e3, 4),
                          "mlups": round(L ** 3 / dt / 1e6), "vs_single": round(dt / base, 4)}), flush=True)
