"""Host envelope refresh (dlb_refresh_envelope_periodic) time on a 512^3 fp32
AcceleratedBlock in pinned memory -- the caller's per-step cost in the e2e
host-block loop."""
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
nbytes = 19 * e ** 3 * 4
p = C.c_void_p()
_capi.check(_capi.lib().dlb_host_alloc(nbytes, C.byref(p)))
blk = np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(p.value)).view(np.float32).reshape(19, e, e, e)
blk[:] = 1.0
for _ in range(2):
    dlb.refresh_envelope_periodic(blk, (1, 1, 1))
t = time.perf_counter()
for _ in range(5):
    dlb.refresh_envelope_periodic(blk, (1, 1, 1))
print(f"refresh_envelope_periodic {L}^3 fp32: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
_capi.lib().dlb_host_free(p)
