"""One e2e configuration on the GPU box: the bench's host-block loop
(refresh_envelope_periodic + collide_and_stream into f_out, pinned, fp32 TGV)
at L^3, 2 warm-up + 6 timed calls; the pipeline knobs come from the
environment (DLB_BLOCK_CHUNKS / DLB_BLOCK_AHEAD / DLB_BLOCK_SPEC), so each
setting runs in its own process: `for a in 1 2 4; do DLB_BLOCK_AHEAD=$a python
tools/e2e_sweep.py 512; done`."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_09242_b200 as dlb  # noqa: E402
from paper_2506_09242_b200 import _capi  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
e = L + 2
reg = dlb.DynamicsRegistry()
slot = reg.register_chain(dlb.init_tgv(dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)).chains[0])
nbytes = 19 * e ** 3 * 4
bufs, keep = [], []
for _ in range(2):
    p = C.c_void_p()
    _capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
    keep.append(p)
    a = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(np.float32).reshape(19, e, e, e)
    a[:] = 0.001
    bufs.append(a)
tag = np.full((e, e, e), -1, np.int32)
tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(slot)
pidx = np.where(tag >= 0, slot, -1).astype(np.int32)
ds = dlb.DispatchSet.all_of(reg)
f = bufs


def step():
    dlb.refresh_envelope_periodic(f[0], (1, 1, 1))
    f[0], f[1] = dlb.collide_and_stream(reg, f[0], tag, pidx, ds, f_out=f[1])


for _ in range(2):
    step()
t = time.perf_counter()
for _ in range(6):
    step()
dt = (time.perf_counter() - t) / 6
knobs = {k: os.environ[k] for k in ("DLB_BLOCK_CHUNKS", "DLB_BLOCK_AHEAD", "DLB_BLOCK_SPEC") if k in os.environ}
print(f"{knobs} {L}^3: {dt * 1e3:.1f} ms/call, {L ** 3 / dt / 1e6:.1f} MLUPS", flush=True)
for p in keep:
    _capi.lib().dlb_host_free(p)
