"""GPU probe: one RQI step (BK factor + solve) at size n (development tool)."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1
n = int(sys.argv[1])
rng = np.random.default_rng(n)
m = rng.standard_normal((n, n)); s = m + m.T
x = rng.standard_normal(n); x /= np.linalg.norm(x)
t0 = time.time(); y = r1.rayleigh_quotient_step(s, x); dt = time.time() - t0
rho = float(x @ (s @ x)); r = s @ y - rho * y; c = float(x @ r)
print(n, "ok", round(dt, 3), np.linalg.norm(r - c * x) / np.linalg.norm(r), flush=True)
