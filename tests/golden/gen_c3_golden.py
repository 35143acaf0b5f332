#!/usr/bin/env python3
"""Golden HOSCF run on BASELINE config 3 (200^4 U(-1,1), 12.8 GB): 100 fixed
iterations (tol 1e-300, record_kkt off: the reference's run_scaling options,
experiment.cpp:195-200), seed 3, from the oracle (oracle/rank1_oracle.py,
pinned to the compiled reference by tests/test_oracle_pins.py).  ~15 CPU
minutes, so the result is committed: tests/golden/c3_hoscf.npz (per-iteration
lambda trace, final lambda and factors).

    python tests/golden/gen_c3_golden.py      # needs ~20 GB of host RAM
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

DIMS = (200, 200, 200, 200)


def main():
    O.build()
    t0 = time.time()
    a = O.gen_config(3, DIMS, 3)
    print(f"generated C3 in {time.time() - t0:.0f} s", flush=True)
    t0 = time.time()
    rep = O.hoscf(a, DIMS, O.Options(tol=1e-300, max_iters=100, seed=3, record_kkt=False))
    print(f"hoscf: {time.time() - t0:.0f} s iterations={rep.iterations} lambda={rep.lam!r}", flush=True)
    out = {"lambda": np.float64(rep.lam), "iterations": np.int64(rep.iterations),
           "trace_lambda": np.array([r["lambda"] for r in rep.trace]),
           "trace_eq11": np.array([r["eq11"] for r in rep.trace])}
    for k, u in enumerate(rep.factors):
        out[f"u{k}"] = np.asarray(u)
    np.savez_compressed(os.path.join(HERE, "c3_hoscf.npz"), **out)
    print("wrote tests/golden/c3_hoscf.npz", flush=True)


if __name__ == "__main__":
    main()
