#!/usr/bin/env python3
"""Randomised check of the tiled grid Lanczos (n > 1024) on block operators of
orders 2-6 with random (incl. tiny, odd) extents against numpy's dense
eigensolver with the reference's pick / sign rules (development tool).
    python tools/eig_fuzz_probe.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
t0 = time.time()
cnt, bad, steps = 0, [], []
while time.time() - t0 < budget:
    d = int(rng.integers(2, 7))
    while True:
        dims = [int(rng.integers(1, 1800)) if rng.random() < 0.3 else int(rng.integers(1, 400)) for _ in range(d)]
        n = sum(dims)
        if 1024 < n <= 2600:
            break
    dims = tuple(dims)
    nb = sum(dims[m] * dims[k] for m in range(d) for k in range(m + 1, d))
    blocks = rng.standard_normal(nb)
    if rng.random() < 0.3:  # a dominant planted direction (fast convergence)
        blocks *= 0.05
    j = r1.SymBlockMatrix(dims, blocks)
    pair, info = r1.eig_blocks(j)
    w, v = np.linalg.eigh(j.dense())
    k = 0 if abs(w[0]) > abs(w[-1]) * (1 + 1e-12) else -1
    vec = v[:, k]
    i = int(np.argmax(np.abs(vec)))
    vec = vec if vec[i] > 0 else -vec
    gap = min(abs(abs(w[0]) - abs(w[-1])), abs(w[-1] - w[-2]), abs(w[1] - w[0])) / max(abs(w[0]), abs(w[-1]))
    ok_v = abs(pair.value - w[k]) <= 1e-12 * abs(w[k])
    ok_x = np.max(np.abs(pair.vector - vec)) <= 1e-8 or gap < 1e-6
    if not (info["converged"] and ok_v and ok_x):
        bad.append((dims, info, pair.value, w[k], np.max(np.abs(pair.vector - vec)), gap))
    steps.append(info["steps"] + 320 * info["restarts"])
    cnt += 1
print(f"eig fuzz: {cnt} operators, {len(bad)} failures in {time.time() - t0:.0f} s; "
      f"Krylov steps median {np.median(steps):.0f}, max {max(steps)}")
for b in bad[:10]:
    print("  ", b)
