"""Development probe: per-iteration iHOSCF trace, device vs reference, on a case
whose RQI accept decisions are near-ties at stagnation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2403_01778_b200 as r1
from oracle import ref, rank1_oracle as O
dims = (7, 5, 9)
a = O.oracle_random_tensor(dims, 11)
got = r1.solve("ihoscf", r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, max_iters=500, seed=1))
want = ref.solve("ihoscf", a, dims, tol=1e-10, max_iters=500, seed=1)
print("iters", got.iterations, want["iterations"])
for k in range(max(got.iterations, want["iterations"])):
    g = got.trace[k] if k < got.iterations else None
    w = want["trace"][k] if k < want["iterations"] else None
    print(k + 1, f"{g.lambda_:.15f} {int(g.rqi_accepted)} {g.lambda_pre_rqi:.15f} {g.eq11_value:.3e}" if g else "-",
          "|", f"{w['lambda_']:.15f} {int(w['rqi_accepted'])} {w['lambda_pre_rqi']:.15f} {w['eq11']:.3e}" if w else "-")
