#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02_bench_final.log 2>&1; tail -c 200 gpurun_out/r02_bench_final.log
timeout 1200 python bench.py --impl reference > gpurun_out/r02_bench_ref_final.log 2>&1; tail -c 300 gpurun_out/r02_bench_ref_final.log
