#!/usr/bin/env python3
"""iHOSCF accept decisions, device vs compiled reference, on one random tensor
(development tool): where the accept patterns first differ, accept counts, and
the rho_y - rho_mid margins of the device run.
    python tools/rqi_accept_probe.py 14x116x51 16"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from oracle import rank1_oracle as O  # noqa: E402
from oracle import ref  # noqa: E402

dims = tuple(int(x) for x in sys.argv[1].split("x"))
seed = int(sys.argv[2])
tseed = int(sys.argv[3]) if len(sys.argv) > 3 else 1234
a = O.oracle_random_tensor(dims, tseed)
rep = r1.solve("ihoscf", r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, max_iters=400, seed=seed))
w = ref.solve("ihoscf", a, dims, tol=1e-10, max_iters=400, seed=seed)
ga = [t.rqi_accepted for t in rep.trace]
ra = [t["rqi_accepted"] for t in w["trace"]]
print(dims, seed, "iters device", rep.iterations, "ref", w["iterations"], "accepts", sum(ga), sum(ra))
first = next((k for k in range(min(len(ga), len(ra))) if ga[k] != ra[k]), None)
print("first accept mismatch at iteration", first)
# margins on the device: accepted lambda = rho_y; rejected: unknown rho_y
lam_pre = np.array([t.lambda_pre_rqi for t in rep.trace])
lam = np.array([t.lambda_ for t in rep.trace])
eq = np.array([t.eq11_value for t in rep.trace])
req = np.array([t["eq11"] for t in w["trace"]])
for k in range(0, min(len(ga), 400), max(1, min(len(ga), 400) // 25)):
    print(f"  it{k+1}: dev acc={ga[k]} eq11={eq[k]:.3e} | ref acc={ra[k] if k < len(ra) else '-'} "
          f"eq11={req[k] if k < len(req) else float('nan'):.3e}  rel(lam-pre)={(abs(lam[k])-abs(lam_pre[k]))/abs(lam[k]):.2e}")
