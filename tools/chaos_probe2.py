#!/usr/bin/env python3
"""Iteration-count sensitivity of stagnating iHOSCF cases: the compiled
reference and the device solver on the same inputs, original and 1-ulp
perturbed (each entry times 1 + {-1,0,1} 2^-52).  Prints JSON lines."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import rank1_oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

import paper_2403_01778_b200 as r1  # noqa: E402

CASES = [("ihoscf", (20, 20, 20), "c1", 1e-10, 1), ("ihoscf", (7, 5, 9), "gauss", 1e-10, 1),
         ("hoscf", (7, 5, 9), "gauss", 1e-10, 1)]
for alg, dims, kind, tol, seed in CASES:
    a = O.gen_config(1, dims, 1) if kind == "c1" else O.oracle_random_tensor(dims, 11)
    rng = np.random.default_rng(0)
    ref_its, gpu_its = [], []
    for t in range(12):
        b = a.copy() if t == 0 else a * (1 + rng.choice([-1, 0, 1], size=a.size) * 2.0 ** -52)
        w = R.solve(alg, b, dims, tol=tol, max_iters=500, seed=seed)
        g = r1.solve(alg, r1.DenseTensor(dims, b), r1.SolveOptions(tol=tol, max_iters=500, seed=seed))
        ref_its.append(w["iterations"])
        gpu_its.append(g.iterations)
    print(json.dumps({"case": [alg, list(dims), kind], "ref": ref_its, "gpu": gpu_its}), flush=True)
