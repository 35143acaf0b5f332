"""GPU probe: the C1 correctness solve (100^3, all-ones init, sigma-change rule)
timing split; run under different R1_EIG_* settings (development tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg, dims = {"C1": (1, (100, 100, 100)), "C4": (4, (60, 60, 60, 60, 60))}[name]
ctx = r1.default_context()
n = int(np.prod(dims))
a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
d = _lib.dims_arr(dims)
_lib.check(_lib.lib().r1_generate_config(ctx.handle, t.handle, cfg, cfg, _lib.u64p(d), len(dims), 0))
if name == "C1":
    o = r1.SolveOptions(tol=1e-300, max_iters=500, seed=cfg, scf_lambda_rtol=1e-12, init="provided",
                        init_factors=[np.ones(k) for k in dims])
else:
    o = r1.SolveOptions(tol=1e-10, max_iters=100, seed=cfg)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = r1.hoscf(t, o, ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name} [{os.environ.get('R1_EIG_GRID', '-')}/{os.environ.get('R1_EIG_SMALL_ONE_CTA', '-')}] "
          f"rep{rep}: {dt*1e3:.1f} ms iters={res.iterations} lambda={res.result.lambda_:.15g} "
          f"eig={res.wall_eig()*1e3:.1f} build={res.wall_build_j()*1e3:.1f} ms", flush=True)
