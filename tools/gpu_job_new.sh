#!/bin/bash
timeout 900 python -m pytest tests/test_sweep_gpu.py -q -x 2>&1 | tail -2
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2403_01778_b200 as r1
ctx=r1.default_context()
for d in [(200,500,3),(136,480,4),(132,1000,2)]: print(d, ctx.sweep_plan_info(d))"
