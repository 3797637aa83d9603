"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck): dense two-population, AA, z-slabs, row and box TMA,
masked / compacted / list porous sweeps, the host-block drop-in, diagnostics
and the fused kinetic energy."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import numpy as np  # noqa: E402

import paper_2506_09242_b200 as dlb  # noqa: E402
from paper_2506_09242_b200.dolb import DeviceRun  # noqa: E402
from test_ragged import ragged_case  # noqa: E402

dims, per = (37, 19, 23), (1, 0, 1)
for kw in ({}, {"layout": "aa"}, {"slabs": 3}, {"tma": True}):
    reg, rec, slot, st = ragged_case(dims, per, 1)
    run = DeviceRun(dims, per, reg, precision=32, **kw)
    run.fill(slot, st)
    run.advance(5)
    run.kinetic_energy()
    print(kw, run.kernel_name(), flush=True)
for kw in ({"skip_nodynamics": True}, {"sparse_lists": True}):
    reg, rec, slot, st = ragged_case(dims, per, 2, nodyn=True)
    run = DeviceRun(dims, per, reg, precision=64, **kw)
    run.fill(slot, st)
    run.advance(5)
    print(kw, run.kernel_name(), flush=True)
cfg = dlb.CaseConfig(kind="tgv", L=24, Re=400.0, Ma=0.1)
run = dlb.build_run(dlb.init_tgv(cfg), precision=64)
assert run.request_kinetic()
run.advance(3)
run.kinetic_energy()
run.enstrophy()
print("fused kinetic energy + enstrophy", flush=True)
run = dlb.build_run(dlb.init_tgv(cfg), precision=32, tma=True)
run.advance(4)
print("tma", run.kernel_name(), flush=True)
# round 2: AA on linked z-slabs (odd steps store into the neighbour's plane),
# the compacted porous sweep, the 128-bit vectorised sweep, the fused
# regularized segment sweep and the multi-slab group graph
import os  # noqa: E402

reg, rec, slot, st = ragged_case(dims, per, 1)
run = DeviceRun(dims, per, reg, precision=32, layout="aa", slabs=3)
run.fill(slot, st)
run.advance(5)
run.gather_populations()
print("aa slabs", run.kernel_name(), flush=True)
reg, rec, slot, st = ragged_case((36, 19, 23), (0, 1, 1), 2, nodyn=True)
os.environ["DLB_POROUS_COMPACT"] = "1"
run = DeviceRun((36, 19, 23), (0, 1, 1), reg, precision=64, skip_nodynamics=True)
run.fill(slot, st)
run.advance(5)
run.gather_populations()
print("compact", run.kernel_name(), flush=True)
del os.environ["DLB_POROUS_COMPACT"]
os.environ["DLB_VEC"] = "1"
reg, rec, slot, st = ragged_case((36, 19, 23), (1, 0, 1), 1)
run = DeviceRun((36, 19, 23), (1, 0, 1), reg, precision=32)
run.fill(slot, st)
run.advance(5)
print("vec", run.kernel_name(), flush=True)
del os.environ["DLB_VEC"]
vox, _ = dlb.sphere_pack((28, 20, 20), radius=3.0, porosity=0.3, seed=5)
cfg = dlb.CaseConfig(kind="porous", L=28, Ma=0.05, collision=dlb.LinkType.TRT, tau=0.8, upstream=4, downstream=4)
run = dlb.build_run(dlb.init_porous(cfg, solid=(vox == 255)), precision=64, skip_nodynamics=True)
run.advance(5)
print("porous fused", run.kernel_name(), flush=True)
os.environ["DLB_GROUP_GRAPH"] = "1"
cfg = dlb.CaseConfig(kind="cavity", L=24, Re=100.0, Ma=0.1)
run = dlb.build_run(dlb.init_cavity(cfg), precision=64, slabs=4)
run.advance(16)
run.gather_populations()
print("group graph", run.kernel_name(), flush=True)
