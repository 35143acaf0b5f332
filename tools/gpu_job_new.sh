#!/bin/bash
# tensor-memory sub-strips: parity on small shapes (threshold forced down), then timing A/B
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
mkdir -p gpurun_out
echo "== quick check =="
R1_SWEEP_NS_MINP=0 timeout 120 python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
import paper_2403_01778_b200 as r1
from oracle import rank1_oracle as o
ctx = r1.default_context()
for dims in ((128, 200, 9), (100, 100, 100), (136, 480, 40), (300, 130, 20), (128, 113, 7), (500, 64, 12), (200, 64, 6, 5), (1000, 300, 5), (72, 500, 11)):
    info = ctx.sweep_plan_info(dims)
    a = o.oracle_random_tensor(dims, 3)
    f = o.oracle_random_unit_factors(dims, 4)
    t = r1.DenseTensor(dims, a)
    got = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    again = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    scale = o.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
    err = np.max(np.abs(got - o.build_j(a, dims, f)) / (scale + 1e-300))
    print(dims, {k: info[k] for k in ("r0", "t1", "G0", "G1", "nra", "K", "ns", "ts", "nseg")}, "relerr %.2e" % err, "repeat identical", bool(np.array_equal(got, again)), flush=True)
    assert err <= 1e-13
print("quick ok")
PY
echo "== parity suites, sub-strips forced =="
R1_SWEEP_NS_MINP=0 timeout 900 python -m pytest tests/test_sweep_gpu.py tests/test_fuzz_gpu.py -q -x 2>&1 | tail -3
for NS in 1 4 1 4; do
  echo "== NS=$NS =="
  R1_SWEEP_NS=$NS timeout 300 python tools/sweep_probe.py C5 C2 300x400x500 --reps 20 2>&1 | grep -v "CTAs" | grep "median" | sed 's/plan={.*nseg.: \([0-9]*\).*} median/nseg \1 median/'
done
