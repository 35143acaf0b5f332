#!/bin/bash
for S in 3 4; do timeout 400 python tools/fork_fuzz_probe.py 150 $S 2>&1 | tail -2 | cut -c1-300; done
