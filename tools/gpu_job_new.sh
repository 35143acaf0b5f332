#!/bin/bash
timeout 600 python tools/stress_probe.py 5 2>&1 | tail -4
timeout 600 python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2403_01778_b200 as r1
from paper_2403_01778_b200 import _lib
ctx = r1.default_context()
for dims in [(1000, 1000, 1000), (200, 200, 200, 200), (500, 2000, 4000)]:
    n = int(np.prod(dims))
    a = torch.empty(n + 2, dtype=torch.float64, device="cuda"); a.uniform_(-1, 1)
    t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx)
    fac = torch.cat([torch.nn.functional.normalize(torch.rand(d, dtype=torch.float64, device="cuda"), dim=0) for d in dims])
    nb = int(sum(dims[m] * dims[k] for m in range(len(dims)) for k in range(m + 1, len(dims))))
    out = [torch.empty(nb, dtype=torch.float64, device="cuda") for _ in range(2)]
    _lib.check(_lib.lib().r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), out[0].data_ptr(), 0))
    bad = 0
    for rep in range(20):
        _lib.check(_lib.lib().r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), out[1].data_ptr(), 0))
        torch.cuda.synchronize()
        bad += int(not torch.equal(out[0], out[1]))
    print(dims, "bit-identical over 20 sweeps" if bad == 0 else f"MISMATCH in {bad} sweeps", flush=True)
    del t, a
    torch.cuda.empty_cache()
PY
