"""GPU probe (development tool): device time of the Bunch-Kaufman factorisation
(r1x_ldlt_time: CUDA events around bk_factor, the matrix restored on the device
outside the timed region) over sizes, optionally over forced panel cluster sizes
(R1_BK_G, development build).  Usage: bk_time_probe.py n [n ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

ctx = r1.default_context()
reps = int(os.environ.get("REPS", "4"))
for n in [int(a) for a in (sys.argv[1:] or ["1000", "3000", "6500"])]:
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, n))
    s = np.asfortranarray(m + m.T).reshape(-1, order="F").copy()
    ms = np.zeros(reps)
    _lib.check(_lib.lib().r1x_ldlt_time(ctx.handle, n, _lib.dptr(s), reps, _lib.dptr(ms)))
    best = ms[1:].min() if reps > 1 else ms[0]
    print(f"n={n} G={os.environ.get('R1_BK_G', 'auto')} factor {best:.3f} ms "
          f"({1e3 * best / n:.2f} us per column) all={np.round(ms, 3).tolist()}", flush=True)
