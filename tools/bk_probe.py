"""GPU probe: the hand-written Bunch-Kaufman factorisation at RQI sizes
(development tool).  Times r1x_ldlt minus its H2D copy via CUDA events is not
possible from Python, so run it under the ncu launch list for the split."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

ctx = r1.default_context()
for n in [int(a) for a in (sys.argv[1:] or ["1000", "3000", "6500"])]:
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, n))
    s = np.asfortranarray(m + m.T).reshape(-1, order="F").copy()
    ipiv = np.empty(n, dtype=np.int32)
    d, sub = np.empty(n), np.empty(n)
    sg, cd = ctypes.c_int(), ctypes.c_double()
    for rep in range(2):
        t0 = time.perf_counter()
        _lib.check(_lib.lib().r1x_ldlt(ctx.handle, n, _lib.dptr(s), ipiv.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                       _lib.dptr(d), _lib.dptr(sub), ctypes.byref(sg), ctypes.byref(cd)))
        print(f"n={n} rep{rep}: {1e3 * (time.perf_counter() - t0):.2f} ms (incl. H2D/D2H of n^2) cond={cd.value:.3e}",
              flush=True)
