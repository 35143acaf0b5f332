"""GPU probe: HOSCF / iHOSCF on device-generated BASELINE configs; prints the
per-iteration phase split (development tool; bench.py is the contract)."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from paper_2403_01778_b200 import _lib  # noqa: E402

CFGS = {"C1": (1, (100, 100, 100)), "C2": (2, (1000, 1000, 1000)), "C3": (3, (200, 200, 200, 200)),
        "C4": (4, (60, 60, 60, 60, 60)), "C5": (5, (500, 2000, 4000))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["C2"])
    ap.add_argument("--alg", default="hoscf,ihoscf")
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--max-iters", type=int, default=100)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    ctx = r1.default_context()
    for nm in args.names:
        cfg, dims = CFGS[nm]
        n = int(np.prod(dims))
        a = torch.empty(n + 2, dtype=torch.float64, device="cuda")
        t = r1.DeviceTensor.wrap(a.data_ptr(), dims, ctx, keepalive=a)
        d = _lib.dims_arr(dims)
        _lib.check(_lib.lib().r1_generate_config(ctx.handle, t.handle, cfg, cfg, _lib.u64p(d), len(dims), 0))
        for alg in args.alg.split(","):
            for rep_i in range(args.reps):
                o = r1.SolveOptions(tol=args.tol, max_iters=args.max_iters, seed=cfg)
                if nm == "C3":
                    o = r1.SolveOptions(tol=1e-300, max_iters=100, seed=cfg, record_kkt=False)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rep = r1.solve(alg, t, o, ctx)
                dt = time.perf_counter() - t0
                print(f"{nm} {alg} rep{rep_i}: {dt*1e3:.2f} ms iters={rep.iterations} sweeps={rep.total_sweeps} "
                      f"conv={rep.converged} lambda={rep.result.lambda_:.15g} build={rep.wall_build_j()*1e3:.2f} "
                      f"eig={rep.wall_eig()*1e3:.2f} other={(rep.wall_total()-rep.wall_build_j()-rep.wall_eig())*1e3:.2f} ms",
                      flush=True)
                if rep_i == args.reps - 1 and rep.iterations <= 12:
                    for k, r in enumerate(rep.trace):
                        print(f"   it{k+1}: lam={r.lambda_:.15g} eq11={r.eq11_value:.3e} rqi={r.rqi_accepted} "
                              f"build={r.t_build_j*1e3:.3f} eig={r.t_eig*1e3:.3f} other={r.t_other*1e3:.3f}")
        del t, a
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
