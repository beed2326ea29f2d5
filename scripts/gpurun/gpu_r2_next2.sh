#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "next2" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_invariance.py -x -q -k "next2" 2>&1 | tail -15
