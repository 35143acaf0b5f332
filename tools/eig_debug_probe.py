#!/usr/bin/env python3
"""Lanczos phase timings (development build, R1_DEBUG_EIG=1) inside HOSCF solves
of a BASELINE config generated on the device: python tools/eig_debug_probe.py C5"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

CFG = {"C1": (1, (100, 100, 100)), "C2": (2, (1000, 1000, 1000)), "C3": (3, (200, 200, 200, 200)),
       "C4": (4, (60, 60, 60, 60, 60)), "C5": (5, (500, 2000, 4000))}
cfg, dims = CFG[sys.argv[1] if len(sys.argv) > 1 else "C5"]
ctx = r1.default_context()
n = int(np.prod(dims))
a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
gd = _lib.dims_arr(dims)
_lib.check(_lib.lib().r1_generate_config(ctx.handle, t.handle, cfg, cfg, _lib.u64p(gd), len(dims), 0))
for alg in ("hoscf",):
    rep = r1.solve(alg, t, r1.SolveOptions(tol=1e-10, max_iters=int(os.environ.get("ITERS", "200")),
                                           seed=cfg), ctx)
    print(alg, rep.iterations, "t_eig", rep.wall_eig(), "t_build_j", rep.wall_build_j(), flush=True)
