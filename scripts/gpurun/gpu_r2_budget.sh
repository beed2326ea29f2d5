#!/bin/bash
# SM budgets: invariance tests, D6 sweeps (pointers / channel split / budgets)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_invariance.py -x -q 2>&1 | tail -5
timeout 1500 python scripts/d6_sweeps.py > gpurun_out/d6_sweeps.log 2>&1; tail -80 gpurun_out/d6_sweeps.log
