#!/bin/bash
timeout 600 python -m pytest tests/test_sweep_gpu.py -q -x -k "deterministic" 2>&1 | tail -2
