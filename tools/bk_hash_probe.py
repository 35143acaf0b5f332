"""GPU probe (development tool): a hash of the Bunch-Kaufman outputs (ipiv, D,
condition) over a fixed set of matrices, to compare kernel variants bit for
bit (run under different development switches and diff the lines)."""
import ctypes
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

ctx = r1.default_context()
for n in [int(a) for a in (sys.argv[1:] or ["33", "200", "700", "1500", "3000", "6500"])]:
    rng = np.random.default_rng(1000 + n)
    m = rng.standard_normal((n, n))
    if n % 2:
        m[:, :5] *= 1e-3  # small columns: interchanges and 2x2 pivots early
    s = np.asfortranarray(m + m.T).reshape(-1, order="F").copy()
    ipiv = np.empty(n, dtype=np.int32)
    d, sub = np.empty(n), np.empty(n)
    sg, cd = ctypes.c_int(), ctypes.c_double()
    _lib.check(_lib.lib().r1x_ldlt(ctx.handle, n, _lib.dptr(s), ipiv.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                   _lib.dptr(d), _lib.dptr(sub), ctypes.byref(sg), ctypes.byref(cd)))
    h = hashlib.sha1(ipiv.tobytes() + d.tobytes() + sub.tobytes() + np.float64(cd.value).tobytes()).hexdigest()[:16]
    print(f"n={n} hash={h} two_by_two={(ipiv < 0).sum()} cond={cd.value:.6e}", flush=True)
