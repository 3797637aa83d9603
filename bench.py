#!/usr/bin/env python3
"""Benchmark of the B200 collide-and-stream path (contract in the task README).

Default workload (N = 1): BASELINE.json config 5 — Taylor-Green vortex, D3Q19
BGK, fp32, 1024^3, Re = 1600, Ma = 0.2 — the largest single-GPU configuration
and the one the north-star target (>= 80 % of the HBM roofline for D3Q19 BGK
on one GPU) is quoted on. Strong scaling: the 1024^3 domain is split into N
z-slabs, one per rank, linked by the fused peer-memory halo push.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
  python bench.py --impl reference ...     # the reference CPU solver (oracle/_ref)

One JSON line is printed by rank 0. `value` is whole-job MLUPS with the state
resident in HBM; `e2e` is the same metric through the reference-facing C ABI
call on HOST buffers (dlb_collide_and_stream: host->device copy of the block,
the step, device->host copy of the new state, every step).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # name: (kind, L, Re, Ma, collision, q, bits, scaling, description)
    "c1": ("cavity", 64, 1000.0, 0.1, "BGK", 19, 64, "strong",
           "lid-driven cavity D3Q19 BGK 64^3 fp64"),
    "c2": ("tgv", 256, 1600.0, 0.2, "RR", 27, 64, "strong",
           "Taylor-Green vortex Re=1600 D3Q27 recursive-regularized 256^3 fp64"),
    "c3": ("cavity", 512, 1000.0, 0.1, "TRT", 19, 32, "weak",
           "lid-driven cavity D3Q19 TRT 512^3 per GPU fp32 (weak scaling)"),
    "c4": ("porous", 600, 0.0, 0.01, "TRT", 19, 64, "strong",
           "synthetic Berea-like porous medium: seeded sphere pack (R=8, ~20% porosity) 600^3 "
           "+ 40/40 fluid buffers, D3Q19 TRT fp64, bounce-back, regularized velocity inlet/outlet"),
    "c5": ("tgv", 1024, 1600.0, 0.2, "BGK", 19, 32, "strong",
           "Taylor-Green vortex D3Q19 BGK 1024^3 fp32 (strong scaling)"),
}


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if "Active" in s[2 + k]
                          and "Not" not in s[2 + k]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_reference(kind, L, Re, Ma, collision, q, bits, warmup, steps, reps=3):
    """The reference CPU solver (oracle/_ref, built from /root/reference) on the
    host cores: N workers x N z-blocks, perf::measure_mlups semantics."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import BGK, RR, TRT, Case, Reference  # checker / baseline only
    if not Reference.available():
        return None
    workers = min(os.cpu_count() or 1, L, 64)
    cid = {"BGK": BGK, "TRT": TRT, "RR": RR}[collision]
    if kind == "porous":
        # same recipe at a bounded size: seeded sphere pack (R=8, 20 %) + 40/40 buffers
        import tempfile

        import paper_2506_09242_b200 as dlb
        vox, _ = dlb.sphere_pack((L, L, L), radius=8.0, porosity=0.20, seed=20250611)
        path = os.path.join(tempfile.gettempdir(), f"dlb_sphere_{L}.raw")
        vox.tofile(path)
        case = Case(kind="porous", L=L, Ma=Ma, collision=cid, tau=1.0, geometry=path,
                    voxel_dims=(L, L, L), upstream=40, downstream=40)
    else:
        case = Case(kind=kind, L=L, Re=Re, Ma=Ma, collision=cid)
    mean, reps_ = Reference().bench(case, bits, workers, warmup, steps, reps)
    return mean, reps_, workers


def run_reference_arm(args, cfgname):
    kind, L, Re, Ma, coll, q, bits, scaling, desc = CONFIGS[cfgname]
    if args.L:
        L = args.L
    rank = env_int("RANK", 0)
    if rank != 0:
        return
    if q != 19:
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no D3Q27 path"}))
        return
    # bounded sample: 512^3 (fp32) / 256^3 (fp64); the full 1024^3 fp32 lattice
    # needs ~187 GB in the reference's block layout (two populations + 16 B of
    # tag / param / cell index per cell, one envelope per worker block), more
    # than the box's host RAM leaves for it
    Ls = min(L, 512 if bits == 32 else 256)
    if kind == "porous":
        Ls = min(L, 256)
    res = cpu_reference(kind, Ls, Re, Ma, coll, q, bits, args.warmup, args.steps, reps=3)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    mean, reps_, workers = res
    sample = (f"{kind} {Ls}^3 D3Q{q} {coll} fp{bits}, {workers} workers x z-blocks, "
              f"warmup {args.warmup} + 3 repetitions x {args.steps} steps, mean (perf::measure_mlups "
              f"semantics, perfmodel.cpp:94-121); per-repetition MLUPS {[round(float(v), 1) for v in reps_]}")
    if Ls < L:
        sample += f"; {Ls}^3 instead of {L}^3: host RAM (the reference's full-size layout does not fit)"
    ms = Ls ** 3 / (mean * 1e6) * 1e3
    line = {
        "impl": "reference", "metric": "MLUPS", "value": mean, "unit": "MLUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32" if bits == 32 else "f64", "data": "synthetic",
        "config": {"workload": f"{cfgname}: {desc}", "sample_L": Ls},
        "cpu_baseline": {"value": mean, "unit": "MLUPS", "cores": workers, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": mean, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def e2e_block(L, bits, steps, warmup, rank=0, world=1, barrier=lambda: None, max_over_ranks=lambda v: v):
    """The same metric through dlb_collide_and_stream on pinned HOST buffers
    (reference-facing drop-in for collide_and_stream(AcceleratedBlock<T>&, ...)):
    per step the caller refreshes the periodic envelope, the call copies the
    block host->device, steps, and copies the new state device->host. With N
    ranks every rank steps its own z-slab block of the L^3 domain (the
    reference's one block per worker) on its GPU; the envelope is refreshed
    from the block itself (the bytes of the host exchange, without the
    transport); the time is the max over ranks."""
    import ctypes as C

    import paper_2506_09242_b200 as dlb
    from paper_2506_09242_b200 import _capi
    from paper_2506_09242_b200.dolb import _Lattice
    cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
    setup = dlb.init_tgv(cfg)
    reg = dlb.DynamicsRegistry()
    slot = reg.register_chain(setup.chains[0])
    dt = np.float32 if bits == 32 else np.float64
    z0, nz = dlb.partition(L, world)[rank]
    ex, ez = L + 2, nz + 2
    nbytes = 19 * ex * ex * ez * np.dtype(dt).itemsize
    p, p2 = C.c_void_p(), C.c_void_p()
    _capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
    _capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p2)))
    try:
        blk = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(dt).reshape(19, ez, ex, ex)
        out = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p2.value)).view(dt).reshape(19, ez, ex, ex)
        out[:] = 0
        # initial state: this block's planes of the TGV state, built on the device
        d = _capi.LatticeDesc()
        d.dims[0], d.dims[1], d.dims[2] = L, L, nz
        for a in range(3):
            d.periodic[a] = 1
        d.q, d.precision_bits, d.arith = 19, bits, _capi.ARITH_EXACT
        d.layout = _capi.LAYOUT_AA if world == 1 else _capi.LAYOUT_TWO_POP  # (AA: single-slab lattices)
        d.device = int(__import__("torch").cuda.current_device())
        d.z_origin, d.global_nz = z0, L
        lat = _Lattice(d, reg)
        _capi.check(_capi.lib().dlb_lattice_set_uniform_slot(lat.handle, slot))
        _capi.check(_capi.lib().dlb_lattice_fill_tgv(lat.handle, L, cfg.lattice_velocity()))
        raw = np.zeros(19 * L * L * nz, dt)
        _capi.check(_capi.lib().dlb_lattice_download_raw(lat.handle, raw.ctypes.data))
        del lat
        blk[:, 1:-1, 1:-1, 1:-1] = raw.reshape(19, nz, L, L)
        del raw
        tag = np.full((ez, ex, ex), -1, np.int32)
        tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(slot)
        pidx = np.where(tag >= 0, slot, -1).astype(np.int32)
        ds = dlb.DispatchSet.all_of(reg)

        f = [blk, out]  # the block's f_in / f_out, swapped by every call (accelerated_lattice.cpp:199)

        def step():
            # refresh_envelope_periodic (accelerated_lattice.cpp:202-238), then the step; C ABI
            dlb.refresh_envelope_periodic(f[0], (1, 1, 1))
            f[0], f[1] = dlb.collide_and_stream(reg, f[0], tag, pidx, ds, f_out=f[1])

        for _ in range(warmup):
            step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            step()
        t1 = time.perf_counter()
        barrier()
        dt_max = max_over_ranks(t1 - t0)
        mlups = L ** 3 * steps / dt_max / 1e6
        d2h_bytes = int(19 * L * L * nz * np.dtype(dt).itemsize)
        link = pcie_ceiling()
        per_rank_gbs = (nbytes + d2h_bytes) * steps / dt_max / 1e9
        return {"value": mlups, "unit": "MLUPS", "h2d_bytes_per_step": int(nbytes) * world,
                "d2h_bytes_per_step": d2h_bytes * world,
                "pcie": {"achieved_gbs_per_gpu": per_rank_gbs, "ceiling_gbs_per_gpu": link,
                         "frac": per_rank_gbs / link if link else None,
                         "ceiling": "1 GiB pinned H2D + D2H copies at once on this GPU, measured in this run"},
                "sample": f"host AcceleratedBlock {L}^3 (+envelope) fp{bits} as {world} z-slab block(s), one per "
                          f"GPU, pinned f_in + f_out swapped per call, {steps} steps, wall clock incl. envelope "
                          "refresh, H2D, step, D2H",
                "finite": bool(np.isfinite(f[0][:, 1:-1, 1:-1, 1:-1]).all())}
    finally:
        _capi.lib().dlb_host_free(p)
        _capi.lib().dlb_host_free(p2)


def pcie_ceiling():
    """Bidirectional host<->device copy rate (GB/s) of this GPU: 1 GiB pinned
    buffers copied both ways at once, best of 3 -- the ceiling of the host-block
    e2e loop, which moves the whole state over PCIe every step."""
    import torch
    n = 1 << 30
    try:
        h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
        d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    except Exception:
        return None
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 0.0
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, 2 * n / (time.perf_counter() - t) / 1e9)
    del h_in, h_out, d_a, d_b
    return best


def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn_ranks(n):
    """--gpus N without a launcher: start N ranks (one process per GPU) with
    torch.distributed.run on this node and pass rank 0's line through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=dict(os.environ, DLB_BENCH_SPAWNED="1"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--L", type=int, default=None,
                    help="edge length at N = 1 (profiling / tests; weak-scaling configs still grow with N)")
    ap.add_argument("--arith", default="exact", choices=["exact", "fast"])
    ap.add_argument("--layout", default="twopop", choices=["twopop", "aa"])
    ap.add_argument("--tma", action="store_true", help="TMA-staged dense kernel instead of the plain-load one")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-L", type=int, default=None, help="edge length of the e2e host-block sample")
    ap.add_argument("--porous", default="masked", choices=["dense", "masked", "lists"],
                    help="c4 kernel variant: dense sweep of every cell (reference behaviour), masked "
                         "sweep (NoDynamics segments skipped), or kind-sorted sparse lists")
    ap.add_argument("--sparse", action="store_true", help="alias of --porous lists")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    if args.impl == "reference":
        run_reference_arm(args, args.config)
        return

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    if world == 1 and args.gpus > 1 and not os.environ.get("DLB_BENCH_SPAWNED"):
        sys.exit(spawn_ranks(args.gpus))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)")

    import torch
    import torch.distributed as tdist

    import paper_2506_09242_b200 as dlb

    local = env_int("LOCAL_RANK", 0)
    same_device = os.environ.get("DLB_SAME_DEVICE") == "1"  # protocol test: all ranks share GPU 0
    if same_device:
        local = 0
    elif torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    # plumbing only (IPC-handle exchange, barriers, the max over ranks): NCCL
    # with one GPU per rank, gloo when the ranks share a device
    backend = "gloo" if same_device else "nccl"
    if world > 1:
        tdist.init_process_group(backend, device_id=None if same_device else torch.device("cuda", local))

    def barrier():
        if world > 1:
            tdist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if same_device else f"cuda:{local}")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    kind, L, Re, Ma, coll, q, bits, scaling, desc = CONFIGS[args.config]
    if args.L:
        L = args.L
    if scaling == "weak":
        L = int(round(L * world ** (1.0 / 3.0)))  # perfmodel.cpp:76-85 weak sizes
    lt = {"BGK": dlb.LinkType.BGK, "TRT": dlb.LinkType.TRT, "RR": dlb.LinkType.RR}[coll]
    skip = False
    extra = {}
    variant = "dense"
    if kind == "porous":
        cfg = dlb.CaseConfig(kind="porous", L=L, Ma=Ma, collision=lt, q=q, tau=1.0, upstream=40,
                             downstream=40)
        vox, phi = dlb.sphere_pack((L, L, L), radius=8.0, porosity=0.20, seed=20250611)
        setup = dlb.init_porous(cfg, solid=(vox == 255))
        kinds = np.bincount(np.asarray(setup.chain_index).reshape(-1), minlength=5)
        variant = "lists" if args.sparse else args.porous
        skip = variant != "dense"
        extra = {"porosity": phi, "fluid_cells": int(kinds[0] + kinds[3] + kinds[4]),
                 "bounce_back_cells": int(kinds[1]), "no_dynamics_cells": int(kinds[2]),
                 "variant": {"lists": "sparse kind-sorted lists (NoDynamics not listed)",
                             "masked": "masked sweep: all-NoDynamics 32-B segments neither loaded nor "
                                       "stored; regularized inlet / outlet cells inside the sweep",
                             "dense": "dense sweep of every cell (regularized planes recomputed by "
                                      "list launches)"}[variant]}
        del vox
    else:
        cfg = dlb.CaseConfig(kind=kind, L=L, Re=Re, Ma=Ma, collision=lt, q=q)
        setup = dlb.init_tgv(cfg) if kind == "tgv" else dlb.init_cavity(cfg)
    layout = args.layout  # AA slabs link like two-population ones (odd steps store across the faces)
    run = dlb.build_run(setup, precision=bits, arith=args.arith,
                        dist=(rank, world) if world > 1 else None, devices=[local], layout=layout,
                        skip_nodynamics=skip, tma=args.tma,
                        sparse_lists=kind == "porous" and variant == "lists")
    del setup
    cells_total = run.num_cells()
    bpc, dev_bytes, launches = run.traffic()
    kernel = run.kernel_name()
    links = dict(run.links(0), rank=rank, device=local, slab_z=list(run.parts[rank]))

    for _ in range(args.warmup):
        run.advance(1)
    run.synchronize()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = run.time_steps(args.steps)  # CUDA events on the lattice stream
        run.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms_max = max_over_ranks(ms)
    ms_step = ms_max / args.steps
    mlups = cells_total * args.steps / (ms_max * 1e-3) / 1e6

    # roofline of the dominant kernel (the fused collide-stream launch(es) of a step)
    my_cells = run.dims[0] * run.dims[1] * sum(p[1] for k, p in enumerate(run.parts) if k in run.ranks)
    peak, peak_kind = measured_peak_hbm()
    alg_bytes = run.step_bytes()  # dense: bytes/cell x cells; sparse: listed links only
    if skip:
        extra["mlups_per_fluid_cell"] = mlups * extra["fluid_cells"] / cells_total
        extra["algorithmic_bytes_per_step"] = alg_bytes
    achieved = alg_bytes / (ms / args.steps * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                tr = json.load(f)
            key = f"{args.config}:{kernel}"
            if key in tr:
                traffic = tr[key]["bytes_per_cell"] * my_cells
        except Exception:
            traffic = None
    all_links = [links]
    if world > 1:
        all_links = [None] * world
        tdist.all_gather_object(all_links, links)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and q == 19:
        Ls = min(L, 256 if (kind == "porous" or bits == 64) else 512)
        res = cpu_reference(kind, Ls, Re, Ma, coll, q, bits, 2, 8, reps=3)
        if res:
            mean, reps_, workers = res
            cpu = {"value": mean, "unit": "MLUPS", "cores": workers, "kind": "reference",
                   "sample": f"{kind} {Ls}^3 D3Q{q} {coll} fp{bits}: reference MultiBlockRun, "
                             f"{workers} workers x z-blocks, warmup 2, 3 reps x 8 steps (mean)"
                             + (f"; {Ls}^3 instead of {L}^3: a bounded sample (host RAM / run time)"
                                if Ls < L else "")}
    e2e = None
    if not args.no_e2e and q == 19 and kind == "tgv":
        del run
        torch.cuda.empty_cache()
        # up to 10 timed calls after 2 warm-up calls (~0.25 s each at 512^3 fp32): the
        # PCIe-bound rate varies by a few percent from call to call
        e2e = e2e_block(args.e2e_L or min(L, 512), bits, max(2, min(args.steps, 10)), 2, rank, world,
                        barrier, max_over_ranks)
    if rank == 0:
        line = {
            "metric": "MLUPS", "value": mlups, "unit": "MLUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if bits == 32 else "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {desc}", "L": L, "cells": cells_total,
                       "parallelism": f"z-slab x{world}",
                       "layout": "AA in-place SoA" if layout == "aa" else "two-population SoA",
                       "arith": args.arith, "kernel": kernel,
                       "l2": "inputs larger than L2 (state resident in HBM)",
                       "device_bytes_per_gpu": dev_bytes,
                       "halo": {"transport": "peer-memory stores from the boundary-plane kernel (CUDA IPC "
                                             "mappings over NVLink), overlapped with the interior launch; "
                                             f"torch.distributed/{backend if world > 1 else '-'} for plumbing",
                                "per_rank": all_links}, **extra},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_cell": bpc},
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    barrier()
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
