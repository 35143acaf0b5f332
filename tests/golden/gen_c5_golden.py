#!/usr/bin/env python3
"""Golden full solves on BASELINE config 5 (reference dims 500 x 2000 x 4000,
32 GB) from the oracle (oracle/rank1_oracle.py: the C restatement of the
sweep and of the Bunch-Kaufman RQI, pinned to the compiled reference by
tests/test_oracle_pins.py; LAPACK eigh for the dense eigenpair).  A full C5
solve takes the CPU oracle ~10-30 minutes, too long for the GPU suite, so the
results are committed: tests/golden/c5_solves.npz (lambda, iterations, the
per-iteration lambda trace and the factors of HOSCF and iHOSCF at tol 1e-10,
seed 5, the options bench.py times).

    python tests/golden/gen_c5_golden.py      # needs ~40 GB of host RAM
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import rank1_oracle as O  # noqa: E402

DIMS = (500, 2000, 4000)


def main():
    O.build()
    t0 = time.time()
    a = O.gen_config(5, DIMS, 5)
    print(f"generated C5 in {time.time() - t0:.0f} s", flush=True)
    out = {}
    for alg in ("hoscf", "ihoscf"):
        t0 = time.time()
        rep = getattr(O, alg)(a, DIMS, O.Options(tol=1e-10, max_iters=200, seed=5))
        print(f"{alg}: {time.time() - t0:.0f} s iterations={rep.iterations} lambda={rep.lam!r} "
              f"converged={rep.converged}", flush=True)
        out[f"{alg}_lambda"] = np.float64(rep.lam)
        out[f"{alg}_iterations"] = np.int64(rep.iterations)
        out[f"{alg}_converged"] = np.bool_(rep.converged)
        out[f"{alg}_trace_lambda"] = np.array([r["lambda"] for r in rep.trace])
        out[f"{alg}_trace_rqi"] = np.array([bool(r["rqi_accepted"]) for r in rep.trace])
        for k, u in enumerate(rep.factors):
            out[f"{alg}_u{k}"] = np.asarray(u)
    np.savez_compressed(os.path.join(HERE, "c5_solves.npz"), **out)
    print("wrote tests/golden/c5_solves.npz", flush=True)


if __name__ == "__main__":
    main()
