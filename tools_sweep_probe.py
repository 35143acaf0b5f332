"""Quick GPU probe: sweep timing at the BASELINE sizes (device-resident input)."""
import sys
import time

import numpy as np
import torch

import paper_2403_01778_b200 as r1
from paper_2403_01778_b200 import _lib

CFGS = {"C2": (1000, 1000, 1000), "C3": (200, 200, 200, 200), "C4": (60, 60, 60, 60, 60),
        "C5": (500, 2000, 4000)}


def run(name, dims, reps=10):
    ctx = r1.default_context()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    n = int(np.prod(dims))
    a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
    a.uniform_(-1, 1)
    t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx)
    fac = torch.cat([torch.nn.functional.normalize(torch.rand(d, dtype=torch.float64, device="cuda"), dim=0) for d in dims])
    nb = int(sum(dims[m] * dims[k] for m in range(len(dims)) for k in range(m + 1, len(dims))))
    blocks = torch.empty(nb, dtype=torch.float64, device="cuda")
    fro = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(3):
        _lib.check(_lib.lib().r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), blocks.data_ptr(), fro.data_ptr()))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(s)
    for i in range(reps):
        _lib.check(_lib.lib().r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(), blocks.data_ptr(), 0))
        ev[i + 1].record(s)
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]
    byts = 8 * n + 8 * nb + 8 * sum(dims)
    med = float(np.median(ms))
    print(f"{name} dims={dims} plan={ctx.sweep_plan_info(dims)} median {med:.3f} ms "
          f"min {min(ms):.3f} -> {byts / med / 1e6:.1f} GB/s", flush=True)
    # parity spot-check vs torch einsum for d=3
    if len(dims) == 3:
        A = a[:n].view(dims[2], dims[1], dims[0])  # reversed (row-major view of col-major)
        u0, u1, u2 = fac[:dims[0]], fac[dims[0]:dims[0] + dims[1]], fac[dims[0] + dims[1]:]
        b01 = torch.einsum("kji,k->ij", A, u2)
        got = blocks[:dims[0] * dims[1]].view(dims[1], dims[0]).t()
        print("   B01 max rel err", float((got - b01).abs().max() / b01.abs().max()), flush=True)
    del t


if __name__ == "__main__":
    names = sys.argv[1:] or list(CFGS)
    for nm in names:
        run(nm, CFGS[nm])
        torch.cuda.empty_cache()
