#!/usr/bin/env python3
"""Per-rank slab sweeps of C5 at 1/2/4/8 ranks, timed on ONE GPU: the device
work each rank of the N-GPU run does per sweep (slab 500 x 2000 x 4000/N of
the C5 tensor, its slice of the last factor), through r1_build_j_device.
Prints JSON lines (the exchange is not included: one GPU here)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

ctx = r1.default_context()
_st = torch.cuda.Stream()
torch.cuda.set_stream(_st)
ctx.set_stream(_st.cuda_stream)
L = _lib.lib()
G = (500, 2000, 4000)
for world in (1, 2, 4, 8):
    dims = (G[0], G[1], G[2] // world)
    n = int(np.prod(dims))
    a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
    t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
    gd = _lib.dims_arr(G)
    _lib.check(L.r1_generate_config(ctx.handle, t.handle, 5, 5, _lib.u64p(gd), 3, 0))
    f = torch.rand(sum(dims), dtype=torch.float64, device="cuda")
    nb = dims[0] * dims[1] + dims[0] * dims[2] + dims[1] * dims[2]
    b = torch.empty(nb, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(5):
        _lib.check(L.r1_build_j_device(ctx.handle, t.handle, f.data_ptr(), b.data_ptr(), None))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    reps = 20
    for _ in range(reps):
        _lib.check(L.r1_build_j_device(ctx.handle, t.handle, f.data_ptr(), b.data_ptr(), None))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    alg = 8 * n + 8 * nb + 8 * sum(dims)
    print(json.dumps({"world": world, "slab": list(dims), "sweep_ms": round(ms, 4),
                      "slab_GBps": round(alg / ms / 1e6, 1)}), flush=True)
    del t, a, b
    torch.cuda.empty_cache()
