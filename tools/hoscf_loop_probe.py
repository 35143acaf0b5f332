#!/usr/bin/env python3
"""HOSCF device-loop probe: C1 (sigma rule, 201 iterations) and C4 / C2 solves,
timed warm, with the loop mode (direct / graph / conditional graph) and the
per-phase totals.  Prints JSON lines."""
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

ctx = r1.default_context()
L = _lib.lib()
for cfg, dims, kw in ((1, (100, 100, 100), dict(tol=1e-300, max_iters=500, init="provided",
                                                 scf_lambda_rtol=1e-12, record_kkt=False)),
                      (4, (60, 60, 60, 60, 60), dict(tol=1e-10, max_iters=100, seed=4)),
                      (2, (1000, 1000, 1000), dict(tol=1e-10, max_iters=100, seed=2)))[
                          :int(os.environ.get("PROBE_NCFG", "3"))]:
    n = int(np.prod(dims))
    a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
    t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
    gd = _lib.dims_arr(dims)
    _lib.check(L.r1_generate_config(ctx.handle, t.handle, cfg, cfg, _lib.u64p(gd), len(dims), 0))
    o = r1.SolveOptions(**{k: v for k, v in kw.items() if k != "init"})
    if kw.get("init") == "provided":
        o.init = "provided"
        o.init_factors = [np.ones(v) for v in dims]
    runs = []
    for _ in range(4):
        torch.cuda.synchronize()
        ts = time.perf_counter()
        rep = r1.solve("hoscf", t, o, ctx)
        torch.cuda.synchronize()
        runs.append(time.perf_counter() - ts)
    mode = ctypes.c_int()
    L.r1x_solver_graph_mode(ctx.handle, ctypes.byref(mode))
    print(json.dumps({"cfg": cfg, "mode": mode.value, "iterations": rep.iterations,
                      "converged": rep.converged, "lambda": rep.result.lambda_,
                      "seconds": [round(x, 5) for x in runs], "t_eig": rep.wall_eig(),
                      "t_build_j": rep.wall_build_j(), "t_total_trace": rep.wall_total(),
                      "factor_change_last": rep.trace[-1].factor_change}), flush=True)
    if os.environ.get("PROBE_TRACE"):
        print(json.dumps({"cfg": cfg, "trace_lambda": [r.lambda_ for r in rep.trace][:40],
                          "trace_eq11": [r.eq11_value for r in rep.trace][:40]}), flush=True)
    del t, a
    torch.cuda.empty_cache()
