timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -v "^\.\+" | grep -v "^\s*$" | head -80 > gpurun_out/fail.txt; tail -3 gpurun_out/fail.txt
