"""Development probe: the dense device eigen path on random symmetric matrices."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2403_01778_b200 as r1
ns = [int(x) for x in sys.argv[1:]] or [10 + 17 * t for t in range(8)]
for n in ns:
    rng = np.random.default_rng((n - 10) // 17)
    m = rng.standard_normal((n, n))
    s = m + m.T
    p = r1.largest_magnitude_eigenpair(s)
    w = np.linalg.eigvalsh(s)
    print(n, p.value, w[0], w[-1], flush=True)
