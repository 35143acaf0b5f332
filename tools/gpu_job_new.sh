#!/bin/bash
R1_BK_TRACE=1 timeout 300 python tools/bk_probe.py 3000 6500 2>&1 | grep "r1 bk\|rep1"
