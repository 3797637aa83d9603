"""Self-linked vs unlinked 1024^3 slab: 3 steps each, for an ncu launch list
(per-kernel durations of the wait / boundary / interior launches)."""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2506_09242_b200 as dlb
from paper_2506_09242_b200 import _capi
L = int(next((a for a in sys.argv[1:] if a.isdigit()), 1024))
LAYOUT = "aa" if "--aa" in sys.argv else "twopop"
cfg = dlb.CaseConfig(kind="tgv", L=L, Re=1600.0, Ma=0.2)
for link in (False, True):
    run = dlb.build_run(dlb.init_tgv(cfg), precision=32, slabs=1, layout=LAYOUT)
    h = run.slabs[0].handle
    if link:
        _capi.check(_capi.lib().dlb_lattice_link_local(h, h))
        if LAYOUT == "aa":  # linking clears an AA slab's state
            run.fill_tgv(L, 0.2 / 3 ** 0.5)
        _capi.check(_capi.lib().dlb_lattice_exchange(h))
    run.advance(3)
    run.synchronize()
    del run
