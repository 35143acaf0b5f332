#!/usr/bin/env python3
"""C1 / C3 HOSCF with the device loop: time, eigen time, iterations and the
lambda trace checksum (development probe for the Lanczos stopping rule)."""
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
for cfg, dims, kw in ((1, (100, 100, 100), dict(tol=1e-300, max_iters=500, scf_lambda_rtol=1e-12, record_kkt=False)),
                      (3, (200, 200, 200, 200), dict(tol=1e-300, max_iters=100, seed=3, record_kkt=False)),
                      (4, (60, 60, 60, 60, 60), dict(tol=1e-10, max_iters=100, seed=4)),
                      (2, (1000, 1000, 1000), dict(tol=1e-10, max_iters=100, seed=2))):
    n = int(np.prod(dims))
    a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
    t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
    gd = _lib.dims_arr(dims)
    _lib.check(_lib.lib().r1_generate_config(ctx.handle, t.handle, cfg, cfg, _lib.u64p(gd), len(dims), 0))
    o = r1.SolveOptions(**kw)
    if cfg == 1:
        o.init = "provided"
        o.init_factors = [np.ones(v) for v in dims]
    for alg in ("hoscf", "ihoscf") if cfg in (2, 4) else ("hoscf",):
        runs = []
        for _ in range(3):
            torch.cuda.synchronize()
            ts = time.perf_counter()
            rep = r1.solve(alg, t, o, ctx)
            torch.cuda.synchronize()
            runs.append(time.perf_counter() - ts)
        lam = np.array([r.lambda_ for r in rep.trace])
        print(json.dumps({"cfg": cfg, "alg": alg, "it": rep.iterations, "s": round(min(runs[1:]), 5),
                          "eig": round(rep.wall_eig(), 5), "lambda": rep.result.lambda_,
                          "trace_sum": float(lam.sum())}), flush=True)
    del t, a
    torch.cuda.empty_cache()
