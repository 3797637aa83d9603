"""Breakdown of the host-block (e2e) path on the GPU box: envelope refresh,
tag scan + step (zero-copy), staged fallback, for one block size."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2506_09242_b200 as dlb
from paper_2506_09242_b200 import _capi

L = int(sys.argv[1]) if len(sys.argv) > 1 else 256
bits = 32
cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
setup = dlb.init_tgv(cfg)
reg = dlb.DynamicsRegistry()
slot = reg.register_chain(setup.chains[0])
e = L + 2
nbytes = 19 * e ** 3 * 4
p = C.c_void_p()
_capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
blk = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(np.float32).reshape(19, e, e, e)
blk[:] = 0
tag = np.full((e, e, e), -1, np.int32)
tag[1:-1, 1:-1, 1:-1] = reg.tag_of_slot(slot)
pidx = np.where(tag >= 0, slot, -1).astype(np.int32)
ds = dlb.DispatchSet.all_of(reg)


def refresh():
    dlb.refresh_envelope_periodic(blk, (1, 1, 1))


def tm(fn, n=3):
    fn()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t) / n


t_ref = tm(refresh)
t_step = tm(lambda: dlb.collide_and_stream(reg, blk, tag, pidx, ds))
pageable = np.zeros((19, e, e, e), np.float32)
t_staged = tm(lambda: dlb.collide_and_stream(reg, pageable, tag, pidx, ds), 2)
n = L ** 3
print(f"L={L} refresh {t_ref*1e3:.1f} ms, zero-copy call {t_step*1e3:.1f} ms ({n/t_step/1e6:.0f} MLUPS), "
      f"staged(pageable) call {t_staged*1e3:.1f} ms ({n/t_staged/1e6:.0f} MLUPS); "
      f"H2D+D2H bytes {2*nbytes/1e9:.2f} GB -> {2*nbytes/t_step/1e9:.1f} GB/s")
_capi.lib().dlb_host_free(p)
