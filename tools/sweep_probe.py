"""GPU probe: sweep timing at the BASELINE sizes (device-resident input), plus a
read/copy bandwidth calibration.  Development tool (bench.py is the contract)."""
import argparse
import time

import numpy as np
import torch

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1
from paper_2403_01778_b200 import _lib

TRACE = False
CFGS = {"C1": (100, 100, 100), "C2": (1000, 1000, 1000), "C3": (200, 200, 200, 200),
        "C4": (60, 60, 60, 60, 60), "C5": (500, 2000, 4000)}


def timeit(fn, s, reps, warm_ms):
    t0 = time.time()
    while (time.time() - t0) * 1e3 < warm_ms:
        fn()
        torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(s)
    for i in range(reps):
        fn()
        ev[i + 1].record(s)
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]


def calib(s, reps, warm_ms):
    n = 1 << 30  # 8 GiB fp64
    a = torch.empty(n, dtype=torch.float64, device="cuda").uniform_()
    ms = timeit(lambda: a.sum(), s, reps, warm_ms)
    print(f"calib torch.sum 8 GiB: median {np.median(ms):.3f} ms -> {8 * n / np.median(ms) / 1e6:.0f} GB/s")
    b = torch.empty(n // 8, dtype=torch.float64, device="cuda")
    c = a[: n // 8]
    ms = timeit(lambda: b.copy_(c), s, reps, warm_ms)
    print(f"calib copy 1 GiB: median {np.median(ms):.3f} ms -> {2 * 8 * n / 8 / np.median(ms) / 1e6:.0f} GB/s")
    del a, b


def run(name, dims, reps, warm_ms, s):
    ctx = r1.default_context()
    ctx.set_stream(s.cuda_stream)
    n = int(np.prod(dims))
    a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
    a.uniform_(-1, 1)
    t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx)
    fac = torch.cat([torch.nn.functional.normalize(torch.rand(d, dtype=torch.float64, device="cuda"), dim=0)
                     for d in dims])
    nb = int(sum(dims[m] * dims[k] for m in range(len(dims)) for k in range(m + 1, len(dims))))
    blocks = torch.empty(nb, dtype=torch.float64, device="cuda")

    def sweep():
        _lib.check(_lib.lib().r1_build_j_device(ctx.handle, t.handle, fac.data_ptr(),
                                                blocks.data_ptr(), 0))

    ms = timeit(sweep, s, reps, warm_ms)
    if TRACE:
        info = ctx.sweep_plan_info(dims)
        tr = torch.zeros(3 * info["ncta"], dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().r1x_set_sweep_trace(ctx.handle, tr.data_ptr()))
        sweep()
        torch.cuda.synchronize()
        _lib.check(_lib.lib().r1x_set_sweep_trace(ctx.handle, None))
        tt = tr.view(-1, 3).cpu().numpy()
        t0 = tt[:, 0].min()
        st = (tt[:, 0] - t0) / 1e3
        en = (tt[:, 1] - t0) / 1e3
        dur = en - st
        print(f"   trace: start max {st.max():.1f} us; end min {en.min():.1f} med {np.median(en):.1f} "
              f"max {en.max():.1f} us; dur min {dur.min():.1f} max {dur.max():.1f}")
        order = np.argsort(en)
        print("   slowest CTAs (cta, smid, end us):", [(int(i), int(tt[i, 2]), round(float(en[i]), 1)) for i in order[-8:]])
        print("   fastest CTAs (cta, smid, end us):", [(int(i), int(tt[i, 2]), round(float(en[i]), 1)) for i in order[:8]])
        np.save(f"gpurun_out/trace_{name}.npy", tt)
    # live per-launch time of the top-level box kernel (CUDA events around it)
    L = _lib.lib()
    import ctypes
    L.r1x_time_kernels(ctx.handle, 1)
    kms, kn = ctypes.c_double(), ctypes.c_uint64()
    L.r1x_kernel_time(ctx.handle, ctypes.byref(kms), ctypes.byref(kn))
    for _ in range(reps):
        sweep()
    torch.cuda.synchronize()
    L.r1x_kernel_time(ctx.handle, ctypes.byref(kms), ctypes.byref(kn))
    L.r1x_time_kernels(ctx.handle, 0)
    print(f"   level-0 box kernel: {kms.value / max(1, kn.value):.4f} ms/launch over {kn.value}")
    byts = 8 * n + 8 * nb + 8 * sum(dims)
    med = float(np.median(ms))
    print(f"{name} dims={dims} plan={ctx.sweep_plan_info(dims)} median {med:.3f} ms "
          f"min {min(ms):.3f} -> {byts / med / 1e6:.1f} GB/s", flush=True)
    del t


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warm-ms", type=float, default=300)
    ap.add_argument("--calib", action="store_true")
    ap.add_argument("--trace", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    TRACE = args.trace
    if args.calib:
        calib(s, args.reps, args.warm_ms)
    for nm in args.names or ["C2", "C3", "C4", "C5"]:
        dims = CFGS[nm] if nm in CFGS else tuple(int(x) for x in nm.split("x"))
        run(nm, dims, args.reps, args.warm_ms, s)
        torch.cuda.empty_cache()
