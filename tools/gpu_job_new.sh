timeout 900 python -m pytest tests/test_sweep_gpu.py -q -x 2>&1 | tail -2
for rep in 1 2; do
echo "== new"; timeout 600 python tools/sweep_probe.py C2 C3 C4 C5 2>&1 | grep -E "^C[0-9]" | sed 's/plan=.*median/median/'
echo "== old"; R1_LIB_PATH=$PWD/_ab/librank1_b200_old.so timeout 600 python tools/sweep_probe.py C2 C3 C4 C5 2>&1 | grep -E "^C[0-9]" | sed 's/plan=.*median/median/'
done
